"""Compact an ncu launch-list CSV (--metrics gpu__time_duration.sum --csv) to
the library's own launches: one line per launch, `id,kernel,grid,block,ns`.

    python scripts/ncu_compact.py in.csv out.csv
"""
import csv
import sys

from launches import UNIT, ours

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
gi, bi, ii = hdr.index("Grid Size"), hdr.index("Block Size"), hdr.index("ID")
with open(sys.argv[2], "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "grid", "block", "ns"])
    for r in rows[1:]:
        if not ours(r[ki]):
            continue
        ns = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0) * 1e6
        w.writerow([r[ii], r[ki].split("(")[0].replace("void ", ""), r[gi], r[bi], "%.0f" % ns])
