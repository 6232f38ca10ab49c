"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel counts, total time and share of the library's own launches.

    python scripts/launches.py launches.csv [--all]

By default only libfrsvt kernels (namespace frsvt / frsvt::tc) are counted:
the bench's synthetic-input generator (torch elementwise kernels) runs
before the timed region and is not part of a step.
"""
import collections
import csv
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3}


def ours(name):
    return name.startswith("void frsvt::") or name.startswith("void tc::") or name.startswith("tc::") \
        or name.startswith("frsvt::")


def summarise(path, only_ours=True, top=40):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1:]:
        name = r[ki]
        if only_ours and not ours(name):
            continue
        short = name.split("(")[0].replace("void ", "")[:70]
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        agg[short][0] += 1
        agg[short][1] += v
        tot += v
    out = ["  share    total ms  launches  avg us   kernel"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append("%6.2f%% %10.3f %8d %9.1f   %s" % (100 * t / tot, t, c, 1e3 * t / c, k))
    out.append("total %.3f ms over %d launches" % (tot, sum(c for c, _ in agg.values())))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], only_ours="--all" not in sys.argv))
