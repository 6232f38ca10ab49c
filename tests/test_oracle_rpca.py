"""Pins for the iALM host (oracle/rpca.py): dual feasibility with the exact
backend, E -> 0 on an uncorrupted low-rank D, exact-vs-FRSVT backend
agreement, recovery of the planted low-rank part, and the c2
trajectory shape the survey probe predicts."""
import numpy as np
import pytest

from oracle import rpca_ialm
from synth import make_config, omega


def _small_instance(m=60, n=40, r=3, frac=0.05, seed=0):
    rng = np.random.default_rng(seed)
    L0 = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    S0 = np.where(rng.random((m, n)) < frac, rng.uniform(-10, 10, (m, n)), 0.0)
    return L0, S0


def test_exact_backend_dual_feasible_and_recovers():
    L0, S0 = _small_instance()
    D = L0 + S0
    out = rpca_ialm(D, 40, 0, 0, None, backend="exact", L0=L0)
    # ||Y_N||_2 <= 1: Y/mu + ... is a subgradient of ||.||_* at L (iALM dual feasibility)
    assert np.linalg.norm(out["Y"], 2) <= 1.0 + 1e-9
    assert out["hist"]["nrmse"][-1] <= 1e-6
    assert np.linalg.norm(out["E"] - S0) <= 1e-5 * np.linalg.norm(S0)


def test_uncorrupted_lowrank_gives_zero_sparse_part():
    """exactly low-rank D with no corruption -> E = 0, L = D (in the
    regime where RPCA identifies (L0, 0); tiny 60x40 instances do not)."""
    rng = np.random.default_rng(1)
    L0 = rng.standard_normal((200, 2)) @ rng.standard_normal((2, 150))
    out = rpca_ialm(L0, 40, 8, 1, lambda k: np.random.default_rng(k).standard_normal((150, 8)))
    assert np.linalg.norm(out["E"]) <= 1e-10 * np.linalg.norm(L0)
    assert np.linalg.norm(out["L"] - L0) <= 1e-10 * np.linalg.norm(L0)


def test_frsvt_backend_matches_exact_backend():
    """S:466 backend equivalence when l >= rank of every SVT argument's kept part."""
    L0, S0 = _small_instance(seed=2)
    D = L0 + S0
    n2 = np.linalg.norm(D, 2)
    ex = rpca_ialm(D, 35, 0, 0, None, backend="exact", norm2=n2)
    fr = rpca_ialm(D, 35, 10, 2, lambda k: np.random.default_rng(k).standard_normal((40, 10)),
                   norm2=n2)
    assert np.linalg.norm(fr["L"] - ex["L"]) <= 1e-6 * np.linalg.norm(ex["L"])
    assert abs(fr["hist"]["r"][-1] - ex["hist"]["r"][-1]) == 0


@pytest.mark.slow
def test_c2_trajectory_shape():
    """BASELINE c2 (1000x1000, l=60, q=1, RP, 30 iterations): r = 0 while tau
    is large, then the planted rank 50; L recovers L0 (survey probe: NRMSE
    8e-7 fp64)."""
    cfg, d = make_config("c2")
    D = d["D"].double().numpy()
    out = rpca_ialm(D, cfg.iters, cfg.l, cfg.q,
                    lambda k: omega(cfg.seed, k, cfg.n, cfg.l).numpy(), L0=d["L0"].numpy())
    r = out["hist"]["r"]
    assert r[:10] == [0] * 10
    assert r[-1] == 50
    assert out["hist"]["nrmse"][-1] <= 1e-5
    assert out["hist"]["resid"][-1] <= 1e-7
