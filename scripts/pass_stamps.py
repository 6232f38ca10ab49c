"""clock64 stamps of the stream-K pass roles (CTA 0) for one pass: where the
pipeline waits. Usage: python scripts/pass_stamps.py kind dbg"""
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

kind, dbg = int(sys.argv[1]), int(sys.argv[2])
m, n, l = 65536, 8192, 120
A = torch.randn((n, m), device="cuda").t()
B = torch.randn((l, n if kind == 0 else m), device="cuda").t()
h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
h.debug_pass(kind, 8 + dbg, A, B)
out = h.debug_pass(kind, 8 + (dbg | 32), A, B)
t = out.t().contiguous().view(-1).view(torch.int64)[: 8 * 4096].cpu().numpy().reshape(8, 4096).astype(np.float64)
nloc = int((t[1] > 0).sum())
t = t[:, :nloc]
t0 = t[0, 0]
names = ["A-prod got emptyA", "conv got fullA", "conv got tempty", "conv arrived tfull", "MMA got tfull",
         "MMA issued", "B-prod got emptyB", "MMA got fullB"]
print("chunks", nloc, "total cycles", t[5, -1] - t0, "per chunk %.0f" % ((t[5, -1] - t0) / nloc))
for e in range(8):
    d = np.diff(t[e])
    print("%-20s per-chunk median %6.0f mean %6.0f p90 %6.0f" % (names[e], np.median(d), d.mean(), np.percentile(d, 90)))
for a, b, lab in ((1, 3, "conv work (fullA->tfull)"), (4, 5, "MMA issue"), (3, 4, "tfull->MMA sees"),
                  (5, 2, "MMA issued->conv sees tempty (i+3)"), (0, 1, "A load latency")):
    if lab.startswith("MMA issued"):
        d = t[2, 3:] - t[5, :-3]
    else:
        d = t[b] - t[a]
    print("%-36s median %6.0f mean %6.0f" % (lab, np.median(d), d.mean()))
print("timeline (cycles rel. to A-prod got emptyA of chunk 400) for chunks 400..407:")
base = t[0, 400]
for i in range(400, 408):
    print(i, " ".join("%7.0f" % (t[e, i] - base) for e in range(8)))
