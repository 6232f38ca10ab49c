# Round-end measurement (run from the repo root on the box): bench line, the
# launch list of the bench command, one ncu --set full capture of the top
# kernels in steady state, the GPU test suite.
T=${1:-r1f}
mkdir -p gpurun_out
python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_status.txt
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/${T}_status.txt
timeout 300 python scripts/rpca_c5_steps.py 24 > gpurun_out/${T}_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"tc_compose2_kernel" -s 18 -c 1 -o gpurun_out/${T}_prof_compose \
  python scripts/rpca_c5_steps.py 24 > gpurun_out/${T}_ncu_full_compose.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"tc_pass2_kernel|eig_jacobi|gram_dmma|chol_inv" -s 60 -c 8 -o gpurun_out/${T}_prof \
  python scripts/rpca_c5_steps.py 24 > gpurun_out/${T}_ncu_full.log 2>&1; echo ncu2=$? >> gpurun_out/${T}_status.txt
cat gpurun_out/${T}_status.txt
