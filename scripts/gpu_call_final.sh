# Round-end measurement (run from the repo root on the box): bench lines of
# every config (e2e + cpu baseline), per-kernel profiles, the launch list of
# the c5 bench command, ncu --set full captures of the c5 step kernels and of
# the streaming kernels of c2, c3, c4 (each ncu command after the same command
# exited 0 without it).
T=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for c in c5 c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c > gpurun_out/${T}_bench_$c.log 2>&1; echo bench_$c=$? >> gpurun_out/${T}_status.txt
done
for c in c5 c4 c2 c3 c1; do timeout 300 python scripts/kprof.py $c 2 > gpurun_out/${T}_kprof_$c.log 2>&1; done
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/${T}_status.txt
timeout 300 python scripts/rpca_c5_steps.py 24 > gpurun_out/${T}_plain.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"tc_compose2_kernel|tc_pass3_kernel|eig_jacobi|gram_dmma|chol_inv" -s 300 -c 14 -o gpurun_out/${T}_prof \
  python scripts/rpca_c5_steps.py 24 > gpurun_out/${T}_ncu_full.log 2>&1; echo ncu2=$? >> gpurun_out/${T}_status.txt
for c in c2 c3 c4; do
  timeout 300 python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/${T}_plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:"tc_compose2_kernel|tc_pass3_kernel" -s 60 -c 10 -o gpurun_out/${T}_prof_$c \
  python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/${T}_ncu_$c.log 2>&1; echo ncu_$c=$? >> gpurun_out/${T}_status.txt
done
cat gpurun_out/${T}_status.txt
# gpurun copies gpurun_out/ back only below 64 MiB: summarise every ncu report
# here (text summary + raw CSV in base units) and drop the reports
for rep in gpurun_out/${T}_prof*.ncu-rep; do
  [ -f "$rep" ] || continue
  b=${rep%.ncu-rep}
  python scripts/ncu_full_summary.py "$rep" > ${b}_summary.txt 2>&1
  ncu -i "$rep" --page raw --csv --print-units base > ${b}_raw.csv 2>/dev/null
  rm -f "$rep"
done
du -sh gpurun_out
