# standard check: GPU tests, bench (no e2e / cpu baseline), per-kernel profile
mkdir -p gpurun_out
T=${1:-std}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests=$? > gpurun_out/${T}_status.txt
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_status.txt
timeout 300 python scripts/kprof.py 10 20 > gpurun_out/${T}_kprof.log 2>&1
cat gpurun_out/${T}_status.txt; tail -2 gpurun_out/${T}_tests.log
tail -n1 gpurun_out/${T}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'])"
head -30 gpurun_out/${T}_kprof.log | grep -v Warn
