# standard check on a GPU box: GPU tests, smoke, bench lines (all configs, no
# e2e / cpu baseline unless FULL=1), per-kernel profile of steady c5 iterations
mkdir -p gpurun_out
T=${1:-std}
CFGS=${CFGS:-"c5 c1 c2 c3 c4"}
EXTRA=${FULL:+}
[ -z "$FULL" ] && EXTRA="--no-e2e --no-cpu-baseline"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${T}_tests.log 2>&1; echo tests=$? > gpurun_out/${T}_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_status.txt
for c in $CFGS; do
  timeout 600 python bench.py --config $c $EXTRA > gpurun_out/${T}_bench_$c.log 2>&1; echo bench_$c=$? >> gpurun_out/${T}_status.txt
done
[ -n "$KPROF" ] && timeout 300 python scripts/kprof.py 10 20 > gpurun_out/${T}_kprof.log 2>&1
cat gpurun_out/${T}_status.txt; tail -3 gpurun_out/${T}_tests.log; tail -2 gpurun_out/${T}_smoke.log
for c in $CFGS; do tail -n1 gpurun_out/${T}_bench_$c.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); r=d['roofline']
    print('$c', '%.2f' % d['value'], d['unit'], 'ms/step %.2f' % d['ms_per_step'], 'dom', r['kind'], 'frac %.3f' % r['frac'], 'unit_frac %.3f' % r['unit_frac'], {k: round(v['frac'], 3) for k, v in r['per_pass'].items()})
except Exception as e: print('$c', 'no line', e)"; done
