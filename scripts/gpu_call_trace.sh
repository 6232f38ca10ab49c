# Jacobi sweep traces (kept rank, revealed rank, sweeps per call/iteration)
# of c2, c4, c5 and a per-kernel profile of c5: bash scripts/gpu_call_trace.sh
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/trace_smi.txt
for c in c2 c4 c5; do timeout 300 python scripts/eig_trace.py $c > gpurun_out/trace_eig_$c.txt 2>&1; done
timeout 300 python scripts/kprof.py c5 2 > gpurun_out/trace_kprof_c5.txt 2>&1
