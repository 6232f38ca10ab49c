"""Pass-kernel bottleneck probe: time tc_pass2 (impl 8 + dbg bits) at c5
shapes with parts of the pipeline disabled (dbg bits: 1 no MMA, 2 no
conversion, 4 no B loads, 8 no bf16 MMAs), for sketch widths l."""
import sys

import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

m, n = 65536, 8192
A = torch.randn((n, m), device="cuda").t()
for l in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "120,24").split(",")]:
    X = torch.randn((l, n), device="cuda").t()
    Q = torch.randn((l, m), device="cuda").t()
    h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
    for kind, B in ((0, X), (1, Q)):
        for dbg in (0, 1, 2, 3, 4, 5, 6, 7, 8):
            ms = h.debug_pass_timed(kind, 8 + dbg, A, B, 10)
            print("l %3d kind %d dbg %d  %.3f ms  %.0f GB/s" % (l, kind, dbg, ms, m * n * 4 / ms / 1e6), flush=True)
    del h
