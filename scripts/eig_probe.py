"""Probe the small-SVD step on real Grams: run c5 (iALM) and c4 (reweighted
WSVT) at full size, and after selected calls time the EIG kernels on the Gram
that call decomposed. Saves the Grams to gpurun_out/eig_grams.npz.

    python scripts/eig_probe.py [impls, e.g. 0,1]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_00296_b200 as P  # noqa: E402
from synth import make_config  # noqa: E402

impls = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1").split(",")]
out = {}
rec = []


def probe(tag, h):
    sig0, UB0, G, sw0, _ = h.debug_small_svd(0, None, 0)
    Gd = G.clone()
    out[tag] = G.double().cpu().numpy()
    for impl in impls:
        sig, UB, _, sw, ms = h.debug_small_svd(impl, Gd, 5)
        e = torch.linalg.eigvalsh(Gd.cpu()).flip(0).clamp(min=0).sqrt()
        err = float((sig.cpu()[:20] - e[:20]).abs().max() / e[0])
        rec.append({"tag": tag, "impl": impl, "sweeps": sw, "ms": ms, "sig_err_top20": err})
        print(json.dumps(rec[-1]), flush=True)


torch.cuda.set_device(0)
cfg, d = make_config("c5", device="cuda")
D = d["D"]
del d
torch.cuda.empty_cache()
m, n = D.shape
h = P.Frsvt(m, n, cfg.l, cfg.q, rp=True, dtype=torch.float32, seed=cfg.seed)
E = torch.empty_like(D)
A = torch.empty_like(D)
L = torch.empty_like(D)
st = h.rpca_state(D, E, A, L, norm2_D=444.46)
for k in range(30):
    h.rpca_step(st)
    if k in (0, 10, 15, 16, 17, 20, 25, 29):
        probe("c5_it%d" % k, h)
del D, E, A, L, h
torch.cuda.empty_cache()

cfg, d = make_config("c4", device="cuda")
Ac = d["A"]
m, n = Ac.shape
h = P.Frsvt(m, n, cfg.l, cfg.q, rp=True, dtype=torch.float32, seed=cfg.seed)
C, eps = 2.0 * np.sqrt(n), 1e-6
for t in range(6):
    h.apply_weighted(Ac, P.W_RECIPROCAL if t == 0 else P.W_REWEIGHTED, C=C, eps=eps)
    probe("c4_call%d" % t, h)
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/eig_grams.npz", **out)
json.dump(rec, open("gpurun_out/eig_probe.json", "w"), indent=1)
