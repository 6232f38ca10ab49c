mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1_smi.txt
for c in c2 c4 c5; do timeout 300 python scripts/eig_trace.py $c > gpurun_out/c1_eig_$c.txt 2>&1; done
timeout 300 python scripts/kprof.py 10 20 > gpurun_out/c1_kprof.txt 2>&1
