# quick GPU check: CMDS is a ;-separated list of python invocations, T the tag
mkdir -p gpurun_out
T=${T:-q}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
if [ -n "$SMOKE" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$? smoke" >> gpurun_out/${T}_status.txt
fi
i=0
IFS=';' read -ra C <<< "$CMDS"
for c in "${C[@]}"; do
  i=$((i+1)); echo "== $c" >> gpurun_out/${T}_out.log
  timeout ${TO:-600} bash -c "$c" >> gpurun_out/${T}_out.log 2>&1; echo "rc=$? $c" >> gpurun_out/${T}_status.txt
done
cat gpurun_out/${T}_status.txt
