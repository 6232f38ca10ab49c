"""GPU parity: libfrsvt (through the C ABI) against the fp64 oracle on the same
seeded inputs. Tolerances (BASELINE north_star): relative Frobenius (SURVEY
Z14 metric) <= 1e-4 in fp32 and <= 1e-10 in fp64."""
import numpy as np
import pytest
import torch

import oracle
from synth import make_config, omega
from tests.gpu_util import cm, np64, z14

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


def _lowrank_plus_noise(m, n, r, noise, seed, decay=1.0):
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((m, r)))[0]
    V = np.linalg.qr(rng.standard_normal((n, r)))[0]
    s = 100.0 * np.logspace(0, -decay, r)
    return (U * s) @ V.T + noise * rng.standard_normal((m, n))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_omega_matches_generator(P, dtype):
    h = P.Frsvt(300, 257, 13, dtype=dtype, seed=12345)
    for call in (0, 5, 77):
        got = np64(h.draw_omega(call))
        exp = omega(12345, call, 257, 13)
        if dtype == torch.float64:
            assert np.max(np.abs(got - exp.numpy()) / np.maximum(np.abs(exp.numpy()), 1e-300)) <= 8e-16
        else:
            e32 = exp.float().double().numpy()
            ulp = np.spacing(np.abs(e32).astype(np.float32)).astype(np.float64)
            assert np.max(np.abs(got - e32) / ulp) <= 1.0


def test_c1_fp64_parity(P):
    """BASELINE c1: 200x100 fp64, l=10, q=1, Omega from the seed."""
    cfg, d = make_config("c1")
    A, L = d["A"], d["L"]
    _, sL, _ = oracle.jacobi_svd(L.numpy())
    tau = 0.5 * sL[4]
    ref = oracle.frsvt(A.numpy(), omega(cfg.seed, 0, cfg.n, cfg.l).numpy(), cfg.l, cfg.q, tau=tau, rp=False)
    h = P.Frsvt(cfg.m, cfg.n, cfg.l, cfg.q, rp=False, dtype=torch.float64, seed=cfg.seed)
    X, info = h.apply(cm(A, torch.float64), tau, info=True)
    assert z14(X, ref.X, A) <= 1e-10
    assert info.r == ref.r == 5
    assert np.allclose(np.array(info.sigma[: ref.s]), ref.sigma, rtol=1e-12)
    Xe, _, _ = oracle.svt_exact(A.numpy(), tau)
    assert z14(X, Xe, A) <= 1e-7


CASES = [
    # m, n, l, q, rank, rp
    (1037, 613, 37, 2, 18, False),
    (517, 1290, 20, 1, 12, False),
    (300, 200, 128, 1, 60, False),
    (2000, 150, 10, 0, 6, False),
    (333, 333, 64, 1, 30, False),
]


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.float64, 1e-10)])
@pytest.mark.parametrize("m,n,l,q,rank,rp", CASES)
def test_single_call_parity(P, m, n, l, q, rank, rp, dtype, tol):
    A = _lowrank_plus_noise(m, n, rank, 1e-2, seed=m + n + l)
    sA = np.linalg.svd(A, compute_uv=False)
    tau = 0.5 * (sA[rank // 2] + sA[rank // 2 + 1])
    Ag = cm(A, dtype)
    A64 = np64(Ag)
    seed = 777 + l
    ref = oracle.frsvt(A64, omega(seed, 0, n, l).numpy(), l, q, tau=tau, rp=rp)
    h = P.Frsvt(m, n, l, q, rp=rp, dtype=dtype, seed=seed)
    X, info = h.apply(Ag, tau, info=True)
    assert z14(X, ref.X, A64) <= tol
    assert info.r == ref.r


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.float64, 1e-10)])
def test_range_propagation_sequence(P, dtype, tol):
    """Free-running and teacher-forced RP over a drifting sequence."""
    m, n, l, q = 700, 450, 24, 1
    rng = np.random.default_rng(4)
    U0, V0 = rng.standard_normal((m, 12)), rng.standard_normal((n, 12))
    G, H = rng.standard_normal((m, 12)), rng.standard_normal((n, 12))
    seed = 99
    h = P.Frsvt(m, n, l, q, rp=True, dtype=dtype, seed=seed)
    ht = P.Frsvt(m, n, l, q, rp=True, dtype=dtype, seed=seed)
    carry = None
    for c in range(6):
        U = np.linalg.qr(U0 + 0.05 * c * G)[0]
        V = np.linalg.qr(V0 + 0.05 * c * H)[0]
        A = (U * np.logspace(1, -1, 12)) @ V.T + 1e-3 * rng.standard_normal((m, n))
        Ag = cm(A, dtype)
        A64 = np64(Ag)
        tau = 0.3
        ref = oracle.frsvt(A64, omega(seed, c, n, l).numpy(), l, q, tau=tau, carry=carry, rp=True)
        X = h.apply(Ag, tau)
        assert z14(X, ref.X, A64) <= tol, c
        # teacher forcing: the oracle's carry, the same call index
        ht.set_carry(None if carry is None else torch.from_numpy(carry))
        ht.set_call_index(c)
        Xt, info = ht.apply(Ag, tau, info=True)
        assert z14(Xt, ref.X, A64) <= tol, c
        assert info.r == ref.r
        carry = ref.carry
    Qt, r = h.get_carry()
    assert r == carry.shape[1]
    Qn = np64(Qt)
    assert np.linalg.norm(Qn.T @ Qn - np.eye(r)) <= (1e-5 if dtype == torch.float32 else 1e-12)
    # same span as the oracle carry
    assert np.linalg.norm(Qn @ (Qn.T @ carry) - carry) <= (1e-3 if dtype == torch.float32 else 1e-9)


def test_weighted_modes(P):
    m, n, l, q = 600, 500, 30, 2
    A = _lowrank_plus_noise(m, n, 20, 0.05, seed=5, decay=0.5)
    Ag = cm(A, torch.float32)
    A64 = np64(Ag)
    seed = 31
    # explicit per-index thresholds (partial-SVT style: keep the first 3 untouched)
    w = np.concatenate([np.zeros(3), np.full(l - 3, 40.0)])
    ref = oracle.frsvt(A64, omega(seed, 0, n, l).numpy(), l, q, w=w, rp=False)
    h = P.Frsvt(m, n, l, q, rp=False, dtype=torch.float32, seed=seed)
    X = h.apply_weighted(Ag, P.W_EXPLICIT, w=w)
    assert z14(X, ref.X, A64) <= 1e-4
    # reciprocal rule, then the reweighted sequence (BASELINE c4 reading Z13)
    C, eps = 2.0 * np.sqrt(n), 1e-6
    seq = oracle.reweighted_wsvt(A64, 5, l, q, C, eps, lambda t: omega(seed, t, n, l).numpy(), rp=True)
    h = P.Frsvt(m, n, l, q, rp=True, dtype=torch.float32, seed=seed)
    for t in range(5):
        X, info = h.apply_weighted(Ag, P.W_RECIPROCAL if t == 0 else P.W_REWEIGHTED, C=C, eps=eps, info=True)
        assert z14(X, seq[t].X, A64) <= 1e-4, t
        assert info.r == seq[t].r


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_edge_cases(P, dtype):
    # zero matrix -> zero output, r = s = 0
    h = P.Frsvt(130, 70, 8, 1, rp=True, dtype=dtype, seed=1)
    Z = torch.zeros((70, 130), dtype=dtype, device="cuda").t()
    X, info = h.apply(Z, 0.5, info=True)
    assert float(X.abs().max()) == 0.0 and info.r == 0 and info.s == 0
    # exactly low rank (rank 3 < l = 12): rank reveal truncates, result = exact SVT
    A = _lowrank_plus_noise(200, 90, 3, 0.0, seed=3)
    Ag = cm(A, dtype)
    A64 = np64(Ag)
    Xe, _, _ = oracle.svt_exact(A64, 5.0)
    h = P.Frsvt(200, 90, 12, 1, rp=False, dtype=dtype, seed=2)
    X, info = h.apply(Ag, 5.0, info=True)
    assert info.s <= 12 and info.r == 3
    assert z14(X, Xe, A64) <= (1e-5 if dtype == torch.float32 else 1e-10)
    # l = min(m, n): the sketch spans everything -> exact SVT
    B = np.random.default_rng(8).standard_normal((40, 24))
    Bg = cm(B, dtype)
    B64 = np64(Bg)
    Xe, _, _ = oracle.svt_exact(B64, 1.5)
    h = P.Frsvt(40, 24, 24, 1, rp=False, dtype=dtype, seed=2)
    X = h.apply(Bg, 1.5)
    assert z14(X, Xe, B64) <= (1e-4 if dtype == torch.float32 else 1e-10)
    # X may alias A
    Bc = Bg.clone()
    h.apply(Bc, 1.5, X=Bc)
    assert z14(Bc, Xe, B64) <= (1e-4 if dtype == torch.float32 else 1e-10)


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.float64, 1e-10)])
@pytest.mark.parametrize("m,n,l,q,rank", [(200, 100, 10, 1, 5), (64, 300, 16, 2, 9), (500, 40, 5, 0, 3),
                                          (33, 17, 1, 1, 1), (150, 100, 16, 3, 12)])
def test_single_cta_path(P, m, n, l, q, rank, dtype, tol):
    """Calls small enough for one SM (no RP, l <= 16) run Algorithm 1 in one
    CTA (batched.cuh): scalar and explicit-weight thresholds against the
    oracle, the flag reports the path, and an RP handle of the same shape
    keeps the multi-kernel path."""
    A = _lowrank_plus_noise(m, n, rank, 1e-2, seed=m * n + l)
    Ag = cm(A, dtype)
    A64 = np64(Ag)
    sA = np.linalg.svd(A64, compute_uv=False)
    tau = 0.5 * (sA[rank - 1] + sA[rank]) if rank < min(m, n) else 0.5 * sA[-1]
    seed = 4242 + l
    Om = omega(seed, 0, n, l).numpy()
    ref = oracle.frsvt(A64, Om, l, q, tau=tau, rp=False)
    h = P.Frsvt(m, n, l, q, rp=False, dtype=dtype, seed=seed)
    X, info = h.apply(Ag, tau, info=True)
    assert info.flags & P.FLAG_SINGLE_CTA
    assert z14(X, ref.X, A64) <= tol
    assert info.r == ref.r and info.s == ref.s
    assert np.allclose(np.array(info.sigma[: ref.s]), ref.sigma, rtol=1e-5 if dtype == torch.float32 else 1e-12)
    # explicit weights: the first two untouched, the rest at tau
    w = np.concatenate([np.zeros(min(2, l)), np.full(l - min(2, l), tau)])
    Om1 = omega(seed, 1, n, l).numpy()
    refw = oracle.frsvt(A64, Om1, l, q, w=w, rp=False)
    Xw, infow = h.apply_weighted(Ag, P.W_EXPLICIT, w=w, info=True)
    assert infow.flags & P.FLAG_SINGLE_CTA
    assert z14(Xw, refw.X, A64) <= tol
    # the same shape with range propagation takes the multi-kernel path
    hr = P.Frsvt(m, n, l, q, rp=True, dtype=dtype, seed=seed)
    Xr, infor = hr.apply(Ag, tau, info=True)
    assert not infor.flags & P.FLAG_SINGLE_CTA
    assert z14(Xr, ref.X, A64) <= tol


def test_nonfinite_is_reported(P):
    h = P.Frsvt(64, 40, 6, 1, rp=False, dtype=torch.float32, seed=1)
    A = torch.randn(40, 64, device="cuda").t()
    A[3, 5] = float("nan")
    with pytest.raises(P.FrsvtError) as e:
        h.apply(A, 0.1, info=True)
    assert e.value.status == 5


def test_deterministic(P):
    A = cm(_lowrank_plus_noise(900, 500, 40, 0.1, seed=11), torch.float32)
    outs = []
    for _ in range(2):
        h = P.Frsvt(900, 500, 60, 2, rp=True, dtype=torch.float32, seed=5)
        X1 = h.apply(A, 1.0).clone()
        X2 = h.apply(A, 1.0).clone()
        outs.append((X1, X2))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
