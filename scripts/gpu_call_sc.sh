mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sc_build.log 2>&1
timeout 120 python scripts/bt_phase.py 200 100 10 1 1 c1 > gpurun_out/sc_phase.log 2>&1
timeout 120 python scripts/bt_phase.py 200 100 10 1 1 >> gpurun_out/sc_phase.log 2>&1
timeout 120 python scripts/bt_phase.py 64 48 10 1 0 >> gpurun_out/sc_phase.log 2>&1
cat gpurun_out/sc_phase.log
