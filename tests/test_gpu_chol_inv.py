"""The explicit CholeskyQR factor kernel (chol_inv.cuh) alone, through the
frsvt_debug_chol_inv hook: for Y with fp64 Gram G, Y T must be an orthonormal
basis of range(Y) (PAPER.md P:130/P:163 QR_CP, reading R4), the same span as
the oracle's pivoted QR; with r > 0 (range propagation, reading
R11) [Q~ | Y Tp] must be orthonormal and span the same space as the oracle's
partial orthogonalisation of Y_p against Q~. Dependent columns are dropped
(zero columns of T, kept rank s)."""
import numpy as np
import pytest
import torch

import oracle
from oracle.frsvt import partial_orthogonalization

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


def _proj(Q):
    return Q @ Q.T


def _handle(P, l):
    return P.Frsvt(4096, 4096, l, 1, dtype=torch.float32, seed=1)


@pytest.mark.parametrize("l", [16, 37, 64, 120, 128])
def test_full_factor_orthonormal_same_span(P, l):
    rng = np.random.default_rng(l)
    m = 3000
    Y = rng.standard_normal((m, l)) * np.logspace(0, -2, l)   # kappa ~ 1e2
    G = Y.T @ Y
    T, s = _handle(P, l).debug_chol_inv(torch.from_numpy(G), 0)
    T = T.double().cpu().numpy()
    assert s == l
    assert np.all(np.tril(T, -1) == 0.0)
    Q = Y @ T
    assert np.linalg.norm(Q.T @ Q - np.eye(l)) <= 1e-5
    Qo = oracle.qr_cp(Y)
    assert np.linalg.norm(_proj(Q) - _proj(Qo), 2) <= 1e-5


@pytest.mark.parametrize("l,r", [(120, 100), (120, 1), (64, 32), (37, 36), (128, 64), (16, 8)])
def test_rp_fresh_block(P, l, r):
    rng = np.random.default_rng(1000 * l + r)
    m, p = 3000, l - r
    Qt = np.linalg.qr(rng.standard_normal((m, r)))[0]
    # fresh samples mostly inside span(Q~), as a warm RP sketch is
    Yp = Qt @ rng.standard_normal((r, p)) + 1e-2 * rng.standard_normal((m, p))
    Y = np.concatenate([Qt, Yp], axis=1)
    G = Y.T @ Y
    T, s = _handle(P, l).debug_chol_inv(torch.from_numpy(G), r)
    T = T.double().cpu().numpy()
    assert s == l
    assert np.all(T[:, p:] == 0.0)
    Qp = Y @ T[:, :p]
    Q = np.concatenate([Qt, Qp], axis=1)
    assert np.linalg.norm(Q.T @ Q - np.eye(l)) <= 1e-5
    Qo = np.concatenate([Qt, partial_orthogonalization(Qt, Yp)], axis=1)
    assert Qo.shape[1] == l
    assert np.linalg.norm(_proj(Q) - _proj(Qo), 2) <= 1e-5


def test_dependent_columns_dropped(P):
    l, r = 40, 20
    rng = np.random.default_rng(7)
    m = 2000
    Qt = np.linalg.qr(rng.standard_normal((m, r)))[0]
    Yp = rng.standard_normal((m, l - r))
    Yp[:, 3] = Qt @ rng.standard_normal(r)              # inside span(Q~)
    Yp[:, 9] = 2.0 * Yp[:, 5] - Qt[:, 0]                # dependent on earlier columns
    Y = np.concatenate([Qt, Yp], axis=1)
    h = _handle(P, l)
    T, s = h.debug_chol_inv(torch.from_numpy(Y.T @ Y), r)
    T = T.double().cpu().numpy()
    assert s == l - 2
    Qp = Y @ T[:, :l - r]
    assert np.all(T[:, 3] == 0.0) and np.all(T[:, 9] == 0.0)
    keep = [j for j in range(l - r) if j not in (3, 9)]
    Q = np.concatenate([Qt, Qp[:, keep]], axis=1)
    assert np.linalg.norm(Q.T @ Q - np.eye(l - 2)) <= 1e-5
    Qo = np.concatenate([Qt, partial_orthogonalization(Qt, Yp)], axis=1)
    assert Qo.shape[1] == l - 2
    assert np.linalg.norm(_proj(Q) - _proj(Qo), 2) <= 1e-5
    # full factorisation of a rank-deficient Y (r = 0): same drops
    Y2 = Y.copy()
    T2, s2 = h.debug_chol_inv(torch.from_numpy(Y2.T @ Y2), 0)
    assert s2 == l - 2
    T2 = T2.double().cpu().numpy()
    assert np.all(T2[:, r + 3] == 0.0) and np.all(T2[:, r + 9] == 0.0)
    Q2 = (Y2 @ T2)[:, [j for j in range(l) if j not in (r + 3, r + 9)]]
    assert np.linalg.norm(Q2.T @ Q2 - np.eye(l - 2)) <= 1e-5


def test_no_fresh_columns(P):
    """r = l (p = 0, pure warm subspace iteration, reading Z6): T = 0, s = l."""
    l = 24
    rng = np.random.default_rng(3)
    Qt = np.linalg.qr(rng.standard_normal((500, l)))[0]
    T, s = _handle(P, l).debug_chol_inv(torch.from_numpy(Qt.T @ Qt), l)
    assert s == l
    assert torch.count_nonzero(T).item() == 0
