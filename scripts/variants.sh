# run pass_parts (dbg 0) + bench for each library variant in tmp_variants/
mkdir -p gpurun_out
cp paper_1509_00296_b200/libfrsvt.so /tmp/lib_base.so
for f in /tmp/lib_base.so tmp_variants/*.so; do
  cp $f paper_1509_00296_b200/libfrsvt.so
  echo "== $f"
  timeout 300 python scripts/pass_parts.py 120,24 2>&1 | grep "dbg 0"
  timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -n1 | cut -c1-110
done
cp /tmp/lib_base.so paper_1509_00296_b200/libfrsvt.so
