"""Per-iteration kept rank and Jacobi sweeps of the small SVD along an iALM
solve (c2/c3/c5) or the reweighted sequence (c4): python scripts/eig_trace.py c5"""
import sys

import torch

sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
import paper_1509_00296_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
stream = torch.cuda.Stream()
W = bench.Workload(P, name, 1, 0, torch.device("cuda", 0), stream, None)
W.estimate_norm2()
h, cfg = W.h, W.cfg
out = []
with torch.cuda.stream(stream):
    if cfg.kind == "rpca":
        s = h.rpca_state(W.inp, W.E, W.A, W.out, rho=W.rho, norm2_D=W.norm2)
        for k in range(cfg.iters):
            h.rpca_step(s, finalize=(k == cfg.iters - 1))
            inf = h.info()
            out.append((k, inf.r, inf.s, inf.sweeps))
    else:
        for t in range(min(cfg.iters, 20)):
            if cfg.kind == "svt":
                h.apply(W.inp, W.tau, X=W.out)
            else:
                h.apply_weighted(W.inp, P.W_RECIPROCAL if t == 0 else P.W_REWEIGHTED, C=cfg.params["C"],
                                 eps=cfg.params["eps"], X=W.out)
            inf = h.info()
            out.append((t, inf.r, inf.s, inf.sweeps))
print(name, "(iter, r, s, sweeps):", out)
