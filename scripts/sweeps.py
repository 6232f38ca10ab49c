"""Jacobi sweeps and kept rank per c5 iALM iteration (steady state)."""
import sys

import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402
from synth import make_config  # noqa: E402

cfg, d = make_config("c5", device="cuda")
D = d["D"]
del d
torch.cuda.empty_cache()
m, n = D.shape
h = P.Frsvt(m, n, cfg.l, cfg.q, rp=True, dtype=torch.float32, seed=cfg.seed)
E, A, L = torch.empty_like(D), torch.empty_like(D), torch.empty_like(D)
st = h.rpca_state(D, E, A, L, norm2_D=447.8)
out = []
for k in range(40):
    h.rpca_step(st)
    inf = h.info()
    out.append("%d:%d/%d/%d" % (k, inf.r, inf.s, inf.sweeps))
print(" ".join(out))
