"""Pins for oracle/frsvt.py (Algorithm 1) against exact SVT and properties the
paper fixes: exactness when rank(A) <= l, Proposition 1
(P:103-111), the shrunk spectrum, the 2-norm-ball bound (Lemma 1), tau = 0
(S:289), RP edge cases, and the weighted variants (fn. 1)."""
import numpy as np
import pytest

from oracle import frsvt, jacobi_svd, reweighted_wsvt, svt_exact, wsvt_exact
from synth import make_config, omega


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _lowrank(m, n, r, seed, spread=1.0):
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((m, r)))[0]
    V = np.linalg.qr(rng.standard_normal((n, r)))[0]
    s = np.linspace(10.0, 10.0 / spread, r)
    return (U * s) @ V.T


@pytest.mark.parametrize("q", [0, 1, 2])
def test_exact_when_rank_le_l(q):
    """rank(A)=5 <= l=7: FRSVT equals the exact Jacobi SVT."""
    A = _lowrank(300, 200, 5, q, spread=3.0)
    Om = np.random.default_rng(100 + q).standard_normal((200, 7))
    tau = 4.5
    X, s, r = svt_exact(A, tau)
    res = frsvt(A, Om, 7, q, tau=tau, rp=False)
    assert res.s == 5
    assert res.r == r
    assert _rel(res.X, X) <= 1e-12


def test_diagonal_input():
    A = np.zeros((40, 30))
    A[0, 0], A[1, 1], A[2, 2] = 5.0, 3.0, 1.0
    Om = np.random.default_rng(1).standard_normal((30, 5))
    res = frsvt(A, Om, 5, 1, tau=2.0, rp=False)
    expect = np.zeros((40, 30))
    expect[0, 0], expect[1, 1] = 3.0, 1.0
    assert np.linalg.norm(res.X - expect) <= 1e-13
    assert res.r == 2 and res.s == 3


@pytest.mark.parametrize("tau_frac", [0.0, 0.3, 0.9])
def test_prop1_and_spectrum(tau_frac):
    """Prop. 1: X = S_tau(Q Q^T A) for the basis FRSVT built; sigma(X) =
    max(sigma(B) - tau, 0); interlacing sigma_i(B) <= sigma_i(A);
    ||P_Q A - X||_2 <= tau (Lemma 1); tau = 0 gives X = Q Q^T A."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((80, 50)) @ np.diag(np.logspace(0, -3, 50)) @ rng.standard_normal((50, 50))
    Om = rng.standard_normal((50, 12))
    sA = np.linalg.svd(A, compute_uv=False)
    tau = tau_frac * sA[4]
    res = frsvt(A, Om, 12, 1, tau=tau, rp=False)
    Q = res.left
    assert np.linalg.norm(Q.T @ Q - np.eye(res.s)) <= 1e-13
    PA = Q @ (Q.T @ A)
    Xp, sB, r = svt_exact(PA, tau)
    assert _rel(res.X, Xp) <= 1e-12
    assert np.allclose(res.sigma, sB[: res.s], rtol=1e-11, atol=1e-13 * sA[0])
    assert np.all(res.sigma <= sA[: res.s] * (1 + 1e-12))
    _, sX, _ = jacobi_svd(res.X)
    assert np.allclose(sX[: res.r], res.sigma[: res.r] - tau, rtol=1e-11)
    assert np.linalg.norm(PA - res.X, 2) <= tau * (1 + 1e-12) + 1e-13 * sA[0]
    if tau == 0.0:
        assert _rel(res.X, PA) <= 1e-12


@pytest.mark.parametrize("cfg_index", [1, 101, 102])
def test_c1_close_to_exact_svt(cfg_index):
    """BASELINE c1 protocol (Fig. 4 NRMSE): FRSVT(l=10,q=1) vs exact
    SVT with tau = 0.5 sigma_5(L). Survey probe: ~6e-9."""
    cfg, d = make_config("c1", cfg_index=cfg_index)
    A, L = d["A"].numpy(), d["L"].numpy()
    _, sL, _ = jacobi_svd(L)
    tau = 0.5 * sL[4]
    X, _, r = svt_exact(A, tau)
    res = frsvt(A, omega(cfg.seed, 0, cfg.n, cfg.l).numpy(), cfg.l, cfg.q, tau=tau, rp=False)
    assert res.r == r == 5
    assert _rel(res.X, X) <= 1e-7


def test_rp_p_zero_uses_carry():
    """p = l - r = 0: Q = Q~, so with q = 0 X = S_tau(Q~ Q~^T A)."""
    rng = np.random.default_rng(8)
    A = rng.standard_normal((60, 40))
    Qt = np.linalg.qr(rng.standard_normal((60, 6)))[0]
    res = frsvt(A, rng.standard_normal((40, 6)), 6, 0, tau=0.5, carry=Qt, rp=True)
    Xp, _, _ = svt_exact(Qt @ (Qt.T @ A), 0.5)
    assert _rel(res.X, Xp) <= 1e-12


def test_rp_carry_spanning_range():
    """Q~ spans range(A): fresh samples add nothing, s = r = rank."""
    A = _lowrank(70, 50, 4, 9)
    U, s, V = jacobi_svd(A)
    Qt = U[:, :4]
    rng = np.random.default_rng(2)
    res = frsvt(A, rng.standard_normal((50, 8)), 8, 1, tau=1.0, carry=Qt, rp=True)
    X, _, _ = svt_exact(A, 1.0)
    assert res.s == 4
    assert _rel(res.X, X) <= 1e-12


def test_rp_sequence_tracks_exact():
    """A slowly rotating rank-6 sequence (the NNM setting of P:179): RP with
    the carried basis matches exact SVT at every call while rank <= l."""
    rng = np.random.default_rng(5)
    U0 = rng.standard_normal((90, 6))
    V0 = rng.standard_normal((60, 6))
    G, H = rng.standard_normal((90, 6)), rng.standard_normal((60, 6))
    carry = None
    rs = []
    for c in range(5):
        U = np.linalg.qr(U0 + 2e-2 * c * G)[0]
        V = np.linalg.qr(V0 + 2e-2 * c * H)[0]
        A = (U * np.linspace(3.0, 0.5 + 0.1 * c, 6)) @ V.T
        res = frsvt(A, rng.standard_normal((60, 10)), 10, 1, tau=0.75, carry=carry, rp=True)
        X, _, r = svt_exact(A, 0.75)
        assert res.r == r
        assert _rel(res.X, X) <= 1e-10
        carry = res.carry
        rs.append(res.r)
    assert rs[0] > 0


def test_weighted_variants():
    rng = np.random.default_rng(6)
    A = _lowrank(50, 40, 6, 6, spread=4.0) + 1e-3 * rng.standard_normal((50, 40))
    Om = rng.standard_normal((40, 10))
    a = frsvt(A, Om, 10, 2, tau=1.5, rp=False)
    b = frsvt(A, Om, 10, 2, w=np.full(10, 1.5), rp=False)
    assert np.linalg.norm(a.X - b.X) <= 1e-14 * np.linalg.norm(a.X)
    # keep-style thresholds on diag(5,3,1): t = (0, 2, 2) -> diag(5,1,0)
    D = np.diag([5.0, 3.0, 1.0])
    res = frsvt(D, np.random.default_rng(1).standard_normal((3, 3)), 3, 0, w=[0, 2, 2], rp=False)
    assert np.allclose(res.X, np.diag([5.0, 1.0, 0.0]), atol=1e-13)
    # reciprocal rule equals the exact WSVT with the same thresholds
    C, eps = 2.0, 1e-6
    res = frsvt(A, Om, 10, 2, C=C, eps=eps, rp=False)
    X, _, _ = wsvt_exact(A, C / (res.sigma + eps))
    assert _rel(res.X, X) <= 1e-9


def test_reweighted_diagonal_recurrence():
    """On a diagonal input the reweighted prox (reading Z13) follows
    sigma <- max(sigma_A - C/(sigma + eps), 0) per component, converging to
    the fixed point (sigma_A - eps + sqrt((sigma_A + eps)^2 - 4C))/2."""
    sA = np.array([12.0, 9.0, 5.0, 3.0, 1.0])
    A = np.zeros((20, 15))
    A[np.arange(5), np.arange(5)] = sA
    C, eps = 4.0, 1e-6
    omf = lambda t: np.random.default_rng(t).standard_normal((15, 8))
    res = reweighted_wsvt(A, 12, 8, 1, C, eps, omf, rp=True)
    sig = sA - C / (sA + eps)
    sig = np.maximum(sig, 0)
    for t in range(1, 12):
        sig = np.maximum(sA - C / (sig + eps), 0.0)
        got = np.zeros(5)
        got[: res[t].r] = res[t].d[: res[t].r]
        assert np.allclose(got, sig, atol=1e-9)
    disc = (sA + eps) ** 2 - 4 * C
    fp = np.where(disc >= 0, (sA - eps + np.sqrt(np.maximum(disc, 0))) / 2, 0)
    assert np.allclose(sig[:3], fp[:3], rtol=1e-6)
