# Round-1 measurement call: bench line, launch list of the bench command, one
# ncu --set full capture of the top kernels (run from the repo root on the box).
set -x
python bench.py > gpurun_out/r1z_bench.log 2>&1; echo bench=$? >> gpurun_out/r1z_status.txt
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r1z_bench_small.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1z_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r1z_ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/r1z_status.txt
timeout 300 python scripts/rpca_c5_steps.py 24 > gpurun_out/r1z_plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tc_compose_kernel|tc_pass2_kernel|eig_jacobi" -s 40 -c 6 -o gpurun_out/r1z_prof python scripts/rpca_c5_steps.py 24 > gpurun_out/r1z_ncu_full.log 2>&1; echo ncu2=$? >> gpurun_out/r1z_status.txt
cat gpurun_out/r1z_status.txt
