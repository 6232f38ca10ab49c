"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel counts, total time and share."""
import collections, csv, sys

def summarise(path, skip=0, top=30):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1 + skip:]:
        name = r[ki].split('(')[0][:80]
        v = float(r[vi].replace(',', ''))
        v *= {'usecond': 1e-3, 'nsecond': 1e-6, 'msecond': 1.0, 'second': 1e3}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append("%7.2f%% %10.3f ms %6d  %s" % (100 * t / tot, t, c, k))
    out.append("total %.3f ms over %d launches" % (tot, sum(c for c, _ in agg.values())))
    return "\n".join(out)

if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0))
