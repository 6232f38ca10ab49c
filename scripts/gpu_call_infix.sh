set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ix_tests.log 2>&1; echo tests=$? >> gpurun_out/ix_status.txt
for v in 0 1; do FRSVT_INFIX=$v timeout 200 python scripts/passbench.py 2 20 > gpurun_out/ix_pass_$v.log 2>&1; done
for v in 0 1; do FRSVT_INFIX=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ix_bench_$v.log 2>&1; echo bench$v=$? >> gpurun_out/ix_status.txt; done
cat gpurun_out/ix_status.txt; tail -3 gpurun_out/ix_tests.log; cat gpurun_out/ix_pass_*.log; tail -1 gpurun_out/ix_bench_*.log | cut -c1-300
