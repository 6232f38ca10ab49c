"""Adaptive rank prediction (AP, §2.3, Eq. (7)) and the
Prop. 4 residual singular value estimate (§3.2) on the GPU against the
oracle (oracle/adaptive.py, oracle/rpca.py with ap=...):
  * free-running iALM with AP: the same sketch-width and kept-rank
    trajectories, recovery error within 1e-3 of the oracle's (north_star bar);
  * varsigma of one FRSVT call against the oracle's estimate from the same
    Omega (the fp64 Gram's Schur complement vs a Householder projection)."""
import numpy as np
import pytest
import torch

import oracle
from oracle.adaptive import sketch_varsigma
from synth import make_config, omega
from tests.gpu_util import cm, np64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


@pytest.mark.parametrize("name,over", [("c2", dict(m=800, n=600, rank=20, l=48, iters=24)),
                                       ("c5", dict(m=6144, n=768, rank=24, l=64, iters=28, var=1.0 / 6144))])
def test_rpca_with_adaptive_rank_against_oracle(P, name, over):
    cfg, d = make_config(name, **over)
    D = cm(d["D"], torch.float32)
    D64 = np64(D)
    L0 = d["L0"].numpy()
    m, n = D.shape
    n2 = oracle.norm2_power(D64)
    h = P.Frsvt(m, n, cfg.l, cfg.q, rp=True, dtype=torch.float32, seed=cfg.seed)
    ap = h.set_adaptive_rank(a=2, rho=0.05)          # b = l, l0 = ceil(0.1 l), jump = ceil(0.05 n)
    ref = oracle.rpca_ialm(D64, cfg.iters, cfg.l, cfg.q, lambda k: omega(cfg.seed, k, n, cfg.l).numpy(), rp=True,
                           norm2=n2, L0=L0, rho=cfg.params["rho"], ap=ap)
    E, A, L = torch.empty_like(D), torch.empty_like(D), torch.empty_like(D)
    st = h.rpca_state(D, E, A, L, rho=cfg.params["rho"], norm2_D=n2)
    l_gpu, r_gpu = [ap["l0"]], []
    for k in range(cfg.iters):
        h.rpca_step(st, finalize=(k == cfg.iters - 1))
        inf = h.info()
        r_gpu.append(inf.r)
        l_gpu.append(inf.l_next)
    hl = ref["hist"]["l"]
    assert hl[0] == ap["l0"] and max(hl) <= cfg.l
    # widths follow Eq. (7) of the GPU's own kept ranks; both trajectories agree
    for k in range(cfg.iters):
        assert l_gpu[k + 1] == min(r_gpu[k] + (2 if r_gpu[k] < l_gpu[k] else ap["rho_n"]), ap["b"])
    assert sum(a != b for a, b in zip(r_gpu, ref["hist"]["r"])) <= 2, (r_gpu, ref["hist"]["r"])
    assert sum(a != b for a, b in zip(l_gpu[:-1], hl)) <= 2, (l_gpu, hl)
    Lg = np64(L)
    assert abs(np.linalg.norm(Lg - L0) / np.linalg.norm(L0) - ref["hist"]["nrmse"][-1]) <= 1e-3
    assert np.linalg.norm(Lg - ref["L"]) <= 1e-3 * np.linalg.norm(ref["L"])


def test_varsigma_against_oracle(P):
    """One FRSVT call (no RP, explicit Omega): the library's varsigma equals the
    oracle's Prop. 4 estimate from the same sketch, and bounds sigma_l(A)."""
    rng = np.random.default_rng(4)
    m, n, l = 1024, 768, 40
    U = np.linalg.qr(rng.standard_normal((m, n)))[0]
    V = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = np.logspace(1, -1, n)
    A64 = ((U * s) @ V.T).astype(np.float32).astype(np.float64)
    Om = omega(21, 0, n, l).numpy()
    h = P.Frsvt(m, n, l, 1, rp=False, dtype=torch.float32, seed=21)
    h.set_omega(cm(torch.from_numpy(Om), torch.float32))
    _, inf = h.apply(cm(torch.from_numpy(A64), torch.float32), float(s[5]), info=True)
    ref = sketch_varsigma(A64, Om, None, 20.0)
    assert abs(inf.varsigma - ref) <= 1e-3 * ref, (inf.varsigma, ref)
    assert inf.varsigma >= s[l - 1]
