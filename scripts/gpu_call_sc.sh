mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bounds.py tests/test_gpu_batched.py -x -q 2>&1 | tail -15 > gpurun_out/sc_tests.log
cat gpurun_out/sc_tests.log
