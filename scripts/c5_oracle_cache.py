"""Cached free-running oracle run of BASELINE c5 (65536 x 8192 fp32 data, fp64
oracle, 40 iALM iterations, l = 120, q = 1, RP): the reference that the
full-size GPU parity test (tests/test_gpu_fullsize.py) compares against.

Calls only oracle/ (and synth/ for the inputs). Writes
tests/golden/c5_oracle.json: ||D||_2 (oracle block power method), mu_0,
lambda, the per-iteration rank / revealed rank / residual / mu / NRMSE(L, L0)
trajectories, ||L||_F, ||E||_F and L, E at 8192 seeded sample positions.
Runtime ~30 min and ~40 GB of host memory (fp64 m x n arrays).
    python scripts/c5_oracle_cache.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from synth import make_config, omega  # noqa: E402

t0 = time.time()
cfg, d = make_config("c5")
D = d["D"].double().numpy()
L0 = np.ascontiguousarray(d["L0"].numpy())
del d
print("inputs %.0f s" % (time.time() - t0), flush=True)
n2 = oracle.norm2_power(D)
print("norm2 %.12g (%.0f s)" % (n2, time.time() - t0), flush=True)
out = oracle.rpca_ialm(D, cfg.iters, cfg.l, cfg.q, lambda k: omega(cfg.seed, k, cfg.n, cfg.l).numpy(), rp=cfg.rp,
                       norm2=n2, L0=L0, rho=cfg.params["rho"])
print("solve %.0f s" % (time.time() - t0), flush=True)
rng = np.random.default_rng(150900296)
ii = rng.integers(0, cfg.m, 8192)
jj = rng.integers(0, cfg.n, 8192)
h = out["hist"]
res = {
    "source": "scripts/c5_oracle_cache.py: oracle.rpca_ialm on synth c5 (seed %d), fp64" % cfg.seed,
    "config": {"m": cfg.m, "n": cfg.n, "l": cfg.l, "q": cfg.q, "rp": cfg.rp, "iters": cfg.iters,
               "rho": cfg.params["rho"]},
    "norm2_D": n2, "mu0": out["mu0"], "lambda": out["lam"],
    "r": [int(x) for x in h["r"]], "s": [int(x) for x in h["s"]], "resid": h["resid"], "mu": h["mu"],
    "nrmse": h["nrmse"],
    "L_fro": float(np.linalg.norm(out["L"])), "E_fro": float(np.linalg.norm(out["E"])),
    "sample_rows": ii.tolist(), "sample_cols": jj.tolist(),
    "L_samples": out["L"][ii, jj].tolist(), "E_samples": out["E"][ii, jj].tolist(),
    "seconds": time.time() - t0,
}
with open(os.path.join(ROOT, "tests", "golden", "c5_oracle.json"), "w") as f:
    json.dump(res, f)
print("r", res["r"])
print("nrmse final %.3e, resid final %.3e, %.0f s" % (res["nrmse"][-1], res["resid"][-1], res["seconds"]))
