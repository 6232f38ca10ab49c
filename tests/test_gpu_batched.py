"""Batched FRSVT of many small matrices (WNNM patch
groups): every matrix of the batch against the oracle's
Algorithm 1 (oracle.frsvt, no range propagation) with the same Omega:
X within the fp32 bar (Z14 <= 1e-4), the kept rank and the kept singular
values; per-matrix thresholds, explicit weights and ragged shapes."""
import numpy as np
import pytest
import torch

import oracle
from synth import omega
from tests.gpu_util import z14

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


def _batch(B, m, n, rank, seed):
    rng = np.random.default_rng(seed)
    A = np.stack([rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)) * rng.uniform(0.5, 2.0)
                  + 0.01 * rng.standard_normal((m, n)) for _ in range(B)]).astype(np.float32)
    return A


def _dev(A):
    # (batch, m, n) with column-major matrices
    return torch.from_numpy(np.ascontiguousarray(A.transpose(0, 2, 1))).cuda().transpose(1, 2)


@pytest.mark.parametrize("B,m,n,l,q,rank", [(64, 64, 48, 10, 1, 5), (33, 37, 29, 8, 2, 3), (8, 200, 120, 16, 1, 12),
                                            (5, 16, 16, 1, 0, 1)])
def test_batched_tau_against_oracle(P, B, m, n, l, q, rank):
    A = _batch(B, m, n, rank, seed=B + m)
    Om = omega(77, 0, n, l).numpy()
    # tau between sigma_rank and sigma_rank+1 of the sketched spectrum (for
    # l = 1, half the single sketched sigma: a one-sample sketch with q = 0 can
    # miss sigma_1 by a large factor, and a tau near the sketched sigma would
    # let d = sigma - tau amplify fp32 rounding)
    def _tau(a):
        sk = oracle.frsvt(a.astype(np.float64), Om, l, q, tau=0.0, rp=False).sigma
        return 0.5 * (sk[rank - 1] + sk[rank]) if l > rank else 0.5 * sk[0]
    taus = np.array([_tau(a) for a in A])
    X, r, sig = P.batched_apply(_dev(A), torch.from_numpy(Om), q=q, tau=torch.from_numpy(taus))
    torch.cuda.synchronize()
    X, r, sig = X.double().cpu().numpy(), r.cpu().numpy(), sig.cpu().numpy()
    for b in range(B):
        ref = oracle.frsvt(A[b].astype(np.float64), Om, l, q, tau=taus[b], rp=False)
        assert z14(X[b], ref.X, A[b].astype(np.float64)) <= 1e-4, b
        assert r[b] == ref.r, b
        assert np.allclose(sig[b, : ref.r], ref.sigma[: ref.r], rtol=1e-5), b


def test_batched_weighted_and_empty(P):
    B, m, n, l = 16, 48, 40, 8
    A = _batch(B, m, n, 4, seed=9)
    Om = omega(78, 0, n, l).numpy()
    w = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 5.0])
    X, r, _ = P.batched_apply(_dev(A), torch.from_numpy(Om), q=1, w=w)
    torch.cuda.synchronize()
    X = X.double().cpu().numpy()
    for b in range(B):
        ref = oracle.frsvt(A[b].astype(np.float64), Om, l, 1, w=w, rp=False)
        assert z14(X[b], ref.X, A[b].astype(np.float64)) <= 1e-4, b
        assert int(r[b]) == ref.r
    Xe, re, _ = P.batched_apply(_dev(A[:0]), torch.from_numpy(Om), q=1, tau=1.0)
    assert Xe.shape[0] == 0 and re.shape[0] == 0


@pytest.mark.parametrize("B,m,n,l,q,rank", [(20, 200, 100, 10, 1, 5), (7, 37, 29, 8, 2, 3)])
def test_batched_fp64_against_oracle(P, B, m, n, l, q, rank):
    """frsvt_batched_apply_f64: BASELINE c1-shaped fp64 matrices (200 x 100,
    l = 10, q = 1) in one launch, each within the fp64 bar (Z14 <= 1e-10)."""
    rng = np.random.default_rng(B + m)
    A = np.stack([rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n))
                  + 0.01 * rng.standard_normal((m, n)) for _ in range(B)])
    Om = omega(79, 0, n, l).numpy()
    taus = np.array([0.5 * np.linalg.svd(a, compute_uv=False)[rank - 1] for a in A])
    Ad = torch.from_numpy(np.ascontiguousarray(A.transpose(0, 2, 1))).cuda().transpose(1, 2)
    X, r, sig = P.batched_apply(Ad, torch.from_numpy(Om), q=q, tau=torch.from_numpy(taus))
    torch.cuda.synchronize()
    assert X.dtype == torch.float64
    X, r, sig = X.cpu().numpy(), r.cpu().numpy(), sig.cpu().numpy()
    for b in range(B):
        ref = oracle.frsvt(A[b], Om, l, q, tau=taus[b], rp=False)
        assert z14(X[b], ref.X, A[b]) <= 1e-10, b
        assert r[b] == ref.r, b
        assert np.allclose(sig[b, : ref.r], ref.sigma[: ref.r], rtol=1e-11), b
