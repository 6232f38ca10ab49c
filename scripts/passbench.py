"""Time the streaming passes alone (c5 shapes): Y = A X and Z = A^T Q with
each route (0 SIMT, 2 CTA-pair tcgen05 exact, 3 span-only), CUDA
events around `reps` back-to-back calls of the C-ABI test hook."""
import sys

import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

m, n, l = 65536, 8192, 120
impls = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
A = torch.randn((n, m), device="cuda").t()
X = torch.randn((l, n), device="cuda").t()
Q = torch.randn((l, m), device="cuda").t()
h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
for kind, B in ((0, X), (1, Q)):
    for impl in impls:
        ms = h.debug_pass_timed(kind, impl, A, B, reps)
        print("kind %d impl %d  %.3f ms  %.0f GB/s (A bytes)" % (kind, impl, ms, m * n * 4 / ms / 1e6), flush=True)
