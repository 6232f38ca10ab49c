mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_chol_inv.py -x -q > gpurun_out/ci_unit.log 2>&1; echo unit=$? >> gpurun_out/ci_status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ci_tests.log 2>&1; echo tests=$? >> gpurun_out/ci_status.txt
for v in 1 4; do FRSVT_FASTCHOL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ci_bench_$v.log 2>&1; echo bench$v=$? >> gpurun_out/ci_status.txt; done
cat gpurun_out/ci_status.txt
