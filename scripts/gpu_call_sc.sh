mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_chol_inv.py tests/test_gpu_rpca.py tests/test_gpu_frsvt.py tests/test_gpu_fullsize.py -x -q -k "not cached" 2>&1 | tail -5 > gpurun_out/sc_tests.log
cat gpurun_out/sc_tests.log
for c in c4 c5; do timeout 300 python scripts/kprof.py $c 2 2>&1 | grep -v -i warn | grep -E "units per step|chol_inv|eig_jacobi"; done
timeout 600 python bench.py --config c5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'], 'e2e', d['e2e'])"
timeout 300 python bench.py --config c3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], 'e2e', d['e2e']['value'])"
