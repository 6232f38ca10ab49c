# bench c5 (per-pass fractions) and the DRAM bytes / duration of the streaming passes of one c5 step under ncu
mkdir -p gpurun_out
T=${T:-np}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 600 python bench.py --config c5 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_pass3_kernel -s 200 -c 12 --csv python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu.csv 2> gpurun_out/${T}_ncu.err
tail -n1 gpurun_out/${T}_bench.log | cut -c1-200
