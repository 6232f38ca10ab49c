# GPU tests (optionally a -k filter) + c5 bench + pass timing
mkdir -p gpurun_out
T=${1:-b}
timeout 1800 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${T}_tests.log 2>&1; echo tests=$? > gpurun_out/${T}_status.txt
timeout 120 python scripts/passbench.py 2,3 5 > gpurun_out/${T}_pass.log 2>&1
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_c5.log 2>&1; echo bench=$? >> gpurun_out/${T}_status.txt
cat gpurun_out/${T}_status.txt; tail -3 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_pass.log | grep -v Warn
tail -n1 gpurun_out/${T}_bench_c5.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('c5', '%.2f' % d['value'], d['unit'], 'ms/step %.2f' % d['ms_per_step'], 'dom', r['kind'], 'frac %.3f' % r['frac'], 'unit_frac %.3f' % r['unit_frac'], {k: round(v['frac'], 3) for k, v in r['per_pass'].items()})"
