"""FRSVT_OPT_TF32_OMEGA (SURVEY 8(f) NEXT-4 'TF32-exact Omega', PAPER.md
P:223-225): every drawn Omega entry rounded to tf32, so the tensor-core sketch
multiplies A by Omega exactly. A different test matrix, not a different
method: the oracle is given the same rounded Omega (synth.omega(tf32=True))
and the GPU result must match it within the fp32 bar (Z14 <= 1e-4)."""
import numpy as np
import pytest
import torch

import oracle
from synth import omega
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


def test_draw_is_the_generator_bit_exact(P):
    h = P.Frsvt(300, 257, 13, dtype=torch.float32, seed=12345, options=P.FRSVT_OPT_TF32_OMEGA)
    for call in (0, 5, 77):
        got = h.draw_omega(call).double().cpu()
        exp = omega(12345, call, 257, 13, tf32=True)
        assert torch.equal(got, exp)
        assert int((h.draw_omega(call).cpu().view(torch.int32) & 0x1FFF).abs().max()) == 0


def test_fp64_handle_rejects_the_option(P):
    with pytest.raises(P.FrsvtError):
        P.Frsvt(300, 257, 13, dtype=torch.float64, seed=1, options=P.FRSVT_OPT_TF32_OMEGA)


@pytest.mark.parametrize("m,n,l,q,rank", [(1037, 613, 37, 2, 18), (300, 200, 128, 1, 60), (2000, 150, 10, 0, 6)])
def test_single_call_parity(P, m, n, l, q, rank):
    A = _lowrank_plus_noise(m, n, rank, 1e-2, seed=m + n + l)
    sA = np.linalg.svd(A, compute_uv=False)
    tau = 0.5 * (sA[rank // 2] + sA[rank // 2 + 1])
    Ag = cm(A, torch.float32)
    A64 = np64(Ag)
    seed = 777 + l
    ref = oracle.frsvt(A64, omega(seed, 0, n, l, tf32=True).numpy(), l, q, tau=tau, rp=False)
    h = P.Frsvt(m, n, l, q, rp=False, dtype=torch.float32, seed=seed, options=P.FRSVT_OPT_TF32_OMEGA)
    X, info = h.apply(Ag, tau, info=True)
    assert z14(X, ref.X, A64) <= 1e-4
    assert info.r == ref.r


def test_range_propagation_sequence(P):
    """RP over a drifting sequence, free-running, with the tf32 Omega on both sides."""
    m, n, l, q = 700, 450, 24, 1
    rng = np.random.default_rng(4)
    U0, V0 = rng.standard_normal((m, 12)), rng.standard_normal((n, 12))
    G, H = rng.standard_normal((m, 12)), rng.standard_normal((n, 12))
    seed = 99
    h = P.Frsvt(m, n, l, q, rp=True, dtype=torch.float32, seed=seed, options=P.FRSVT_OPT_TF32_OMEGA)
    carry = None
    for c in range(6):
        U = np.linalg.qr(U0 + 0.05 * c * G)[0]
        V = np.linalg.qr(V0 + 0.05 * c * H)[0]
        A = (U * np.logspace(1, -1, 12)) @ V.T + 1e-3 * rng.standard_normal((m, n))
        Ag = cm(A, torch.float32)
        A64 = np64(Ag)
        ref = oracle.frsvt(A64, omega(seed, c, n, l, tf32=True).numpy(), l, q, tau=0.3, carry=carry, rp=True)
        X, info = h.apply(Ag, 0.3, info=True)
        assert z14(X, ref.X, A64) <= 1e-4, c
        assert info.r == ref.r
        carry = ref.carry


def test_reweighted_sequence(P):
    """BASELINE c4's reweighted WSVT (reading Z13) on a small matrix, tf32 Omega."""
    m, n, l, q = 600, 500, 30, 2
    A = _lowrank_plus_noise(m, n, 20, 0.05, seed=5, decay=0.5)
    Ag = cm(A, torch.float32)
    A64 = np64(Ag)
    seed = 31
    C, eps = 2.0 * np.sqrt(n), 1e-6
    seq = oracle.reweighted_wsvt(A64, 5, l, q, C, eps, lambda t: omega(seed, t, n, l, tf32=True).numpy(), rp=True)
    h = P.Frsvt(m, n, l, q, rp=True, dtype=torch.float32, seed=seed, options=P.FRSVT_OPT_TF32_OMEGA)
    for t in range(5):
        X = h.apply_weighted(Ag, P.W_RECIPROCAL if t == 0 else P.W_REWEIGHTED, C=C, eps=eps)
        assert z14(X, seq[t].X, A64) <= 1e-4, t
