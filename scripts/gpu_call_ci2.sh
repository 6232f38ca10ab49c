mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_chol_inv.py -x -q > gpurun_out/ci2_unit.log 2>&1; echo unit=$? >> gpurun_out/ci2_status.txt
timeout 200 python scripts/ci_bench.py > gpurun_out/ci2_cib.log 2>&1
timeout 300 python scripts/kprof.py 2 20 --seq > gpurun_out/ci2_kprof.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ci2_tests.log 2>&1; echo tests=$? >> gpurun_out/ci2_status.txt
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ci2_bench.log 2>&1; echo bench=$? >> gpurun_out/ci2_status.txt
cat gpurun_out/ci2_status.txt
