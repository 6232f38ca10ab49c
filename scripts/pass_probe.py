"""Pipeline probe of the streaming pass at the c5 shape: the exact CTA-pair
pass with parts of its pipeline switched off (impl 8 + dbg; dbg bits: 1 no
MMA, 2 no conversion, 4 no B loads, 16 no accumulator reads). Prints ms and
GB/s of A per variant."""
import sys

import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

m, n, l = 65536, 8192, int(sys.argv[1]) if len(sys.argv) > 1 else 120
A = torch.randn((n, m), device="cuda").t()
X = torch.randn((l, n), device="cuda").t()
Q = torch.randn((l, m), device="cuda").t()
h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
for kind, B in ((0, X), (1, Q)):
    for base, name in ((8, "pass3"),):
        for dbg in (0, 1, 2, 3, 4, 5, 6, 16):
            ms = h.debug_pass_timed(kind, base + dbg, A, B, 10)
            print("kind %d %s dbg %d  %.3f ms  %.0f GB/s" % (kind, name, dbg, ms, m * n * 4 / ms / 1e6), flush=True)
