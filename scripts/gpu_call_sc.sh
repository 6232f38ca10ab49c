mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -k "not cached" 2>&1 | tail -5 > gpurun_out/sc_tests.log
cat gpurun_out/sc_tests.log
for c in c3; do timeout 300 python scripts/kprof.py $c 2 2>&1 | grep -v -i warn | head -8; done
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 3 --warmup 3 --no-e2e 2>&1 | tail -1 | cut -c1-200
