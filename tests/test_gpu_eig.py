"""The small-SVD kernel (Alg. 1 lines 16-18, reading Z8) alone, through the
frsvt_debug_small_svd hook: sigma and U_B of an l x l fp64 Gram G = B B^T
against numpy's symmetric eigensolver, on synthetic spectra shaped like the
iALM Grams (a clustered signal block + a tiny noise block), rank-deficient
Grams and every l class (1 .. 4 rows per lane, odd l)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


def _gram(l, kind, seed):
    rng = np.random.default_rng(seed)
    Q = np.linalg.qr(rng.standard_normal((l, l)))[0]
    if kind == "cluster":      # 5/6 of the spectrum in [0.3, 0.4], the rest ~1e-3
        k = (5 * l) // 6
        s = np.concatenate([rng.uniform(0.3, 0.4, k), rng.uniform(6e-4, 8e-4, l - k)])
    elif kind == "graded":
        s = np.logspace(2, -4, l)
    elif kind == "deficient":  # rank l/2, exact zeros
        s = np.concatenate([rng.uniform(1, 10, l // 2), np.zeros(l - l // 2)])
    else:
        s = rng.uniform(0.5, 2.0, l)
    # nearly diagonal in this basis, as a warm RP Gram is: small random rotation
    if kind == "cluster":
        Kr = 0.02 * rng.standard_normal((l, l))
        Q = np.linalg.qr(np.eye(l) + Kr - Kr.T)[0]
    G = (Q * s**2) @ Q.T
    return 0.5 * (G + G.T), s


@pytest.mark.parametrize("impl", [0])
@pytest.mark.parametrize("l", [10, 37, 64, 120, 128])
@pytest.mark.parametrize("kind", ["cluster", "graded", "deficient", "random"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_small_svd_kernel(P, impl, l, kind, dtype):
    G, s = _gram(l, kind, seed=l + len(kind))
    h = P.Frsvt(max(l, 200), max(l, 150), l, 1, dtype=dtype, seed=1)
    sig, UB, Gc, sweeps, _ = h.debug_small_svd(impl, torch.from_numpy(G))
    sig, UB = sig.cpu().numpy(), UB.cpu().numpy()
    assert np.array_equal(Gc.cpu().numpy(), G)
    e = np.sqrt(np.maximum(np.linalg.eigvalsh(G)[::-1], 0.0))
    assert np.all(np.diff(sig) <= 0.0)
    # sigma: absolute accuracy relative to sigma_1^2 / sigma_i (Gram route)
    tol = 1e-13 if dtype == torch.float64 else 1e-9
    err = np.abs(sig - e) * np.maximum(sig, 1e-300) / e[0] ** 2
    assert err.max() <= tol, err.max()
    # U_B diagonalises G on the non-null part, orthonormal columns there
    keep = sig > 1e-6 * sig[0]
    U = UB[:, keep]
    R = G @ U - U * sig[keep] ** 2
    assert np.linalg.norm(R) <= (1e-12 if dtype == torch.float64 else 1e-8) * e[0] ** 2 * np.sqrt(l)
    assert np.linalg.norm(U.T @ U - np.eye(U.shape[1])) <= (1e-12 if dtype == torch.float64 else 1e-7) * l
    assert 1 <= sweeps < 40
