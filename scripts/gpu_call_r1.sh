set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r1_status.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r1_status.txt
timeout 600 python bench.py > gpurun_out/r1_bench.log 2>&1; echo bench=$? >> gpurun_out/r1_status.txt
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r1_bench_small.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r1_ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/r1_status.txt
timeout 300 python scripts/rpca_c5_steps.py 20 > gpurun_out/r1_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_ -s 20 -c 6 -o gpurun_out/r1_prof python scripts/rpca_c5_steps.py 20 > gpurun_out/r1_ncu_full.log 2>&1; echo ncu2=$? >> gpurun_out/r1_status.txt
cat gpurun_out/r1_status.txt
