"""Pins for oracle/linalg.py against what mathematics fixes independently of
the oracle's own code: closed forms, characteristic polynomials, invariants,
and library routines on special cases."""
import numpy as np
import pytest

from oracle import jacobi_svd, norm2_power, polar_newton, qr_cp


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_jacobi_closed_forms():
    U, s, V = jacobi_svd(np.diag([3.0, 1.0]))
    assert np.allclose(s, [3, 1], atol=1e-15)
    U, s, V = jacobi_svd(np.zeros((4, 3)))
    assert np.all(s == 0)
    assert np.allclose(U.T @ U, np.eye(3), atol=1e-14)
    # scaled rotation: both singular values equal 2
    th = 0.3
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    _, s, _ = jacobi_svd(2 * R)
    assert np.allclose(s, [2, 2], atol=1e-14)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_jacobi_2x2_quadratic(seed):
    """sigma^2 are the roots of lambda^2 - tr(M^T M) lambda + det(M)^2."""
    M = np.random.default_rng(seed).standard_normal((2, 2))
    tr = np.sum(M * M)
    det = M[0, 0] * M[1, 1] - M[0, 1] * M[1, 0]
    disc = np.sqrt(tr * tr - 4 * det * det)
    expect = np.sqrt([(tr + disc) / 2, (tr - disc) / 2])
    _, s, _ = jacobi_svd(M)
    assert np.allclose(s, expect, rtol=1e-13)


@pytest.mark.parametrize("seed", [0, 1])
def test_jacobi_3x3_cubic(seed):
    """sigma^2 are the roots of the characteristic cubic of G = M^T M:
    lambda^3 - c2 lambda^2 + c1 lambda - c0 with c2 = tr G, c1 = sum of the
    principal 2x2 minors, c0 = det(M)^2."""
    M = np.random.default_rng(10 + seed).standard_normal((3, 3))
    G = M.T @ M
    c2 = np.trace(G)
    c1 = (G[0, 0] * G[1, 1] - G[0, 1] ** 2 + G[0, 0] * G[2, 2] - G[0, 2] ** 2
          + G[1, 1] * G[2, 2] - G[1, 2] ** 2)
    detM = (M[0, 0] * (M[1, 1] * M[2, 2] - M[1, 2] * M[2, 1])
            - M[0, 1] * (M[1, 0] * M[2, 2] - M[1, 2] * M[2, 0])
            + M[0, 2] * (M[1, 0] * M[2, 1] - M[1, 1] * M[2, 0]))
    roots = np.sort(np.real(np.roots([1.0, -c2, c1, -detM ** 2])))[::-1]
    _, s, _ = jacobi_svd(M)
    assert np.allclose(s ** 2, roots, rtol=1e-10)


@pytest.mark.parametrize("shape", [(30, 20), (20, 30), (17, 17)])
def test_jacobi_invariants_and_library(shape):
    M = np.random.default_rng(5).standard_normal(shape)
    U, s, V = jacobi_svd(M)
    k = min(shape)
    assert U.shape == (shape[0], k) and V.shape == (shape[1], k)
    assert _rel((U * s) @ V.T, M) <= 1e-13
    assert np.linalg.norm(U.T @ U - np.eye(k)) <= 1e-13
    assert np.linalg.norm(V.T @ V - np.eye(k)) <= 1e-13
    assert np.all(np.diff(s) <= 0)
    assert np.allclose(s, np.linalg.svd(M, compute_uv=False), rtol=1e-12)


def test_jacobi_rank_deficient():
    """a rank-2 30x20 matrix has sigma_3 <= 1e-10 sigma_1."""
    rng = np.random.default_rng(3)
    M = rng.standard_normal((30, 2)) @ rng.standard_normal((2, 20))
    U, s, V = jacobi_svd(M)
    assert s[2] <= 1e-10 * s[0]
    assert np.linalg.norm(U.T @ U - np.eye(20)) <= 1e-12
    assert _rel((U * s) @ V.T, M) <= 1e-13


@pytest.mark.parametrize("cond", [1e1, 1e8])
def test_polar_newton(cond):
    """Definition 2: C = W P, W^T W = I, P symmetric PSD with P^2 = C^T C;
    P:195 'typically, seven' iterations (S:579 allows <= 20)."""
    rng = np.random.default_rng(int(cond))
    Q1 = np.linalg.qr(rng.standard_normal((20, 20)))[0]
    Q2 = np.linalg.qr(rng.standard_normal((20, 20)))[0]
    C = (Q1 * np.logspace(0, -np.log10(cond), 20)) @ Q2.T
    W, P, it = polar_newton(C)
    assert it <= 20
    assert np.linalg.norm(W.T @ W - np.eye(20)) <= 1e-12
    assert np.allclose(P, P.T)
    assert np.min(np.linalg.eigvalsh(P)) >= -1e-14
    assert _rel(W @ P, C) <= 1e-12
    assert _rel(P @ P, C.T @ C) <= 1e-10
    # the polar factor of Q1 S Q2^T is Q1 Q2^T
    assert np.linalg.norm(W - Q1 @ Q2.T) <= 1e-12 * cond


def test_qr_cp_rank_reveal():
    rng = np.random.default_rng(4)
    Y = rng.standard_normal((50, 3)) @ rng.standard_normal((3, 6))
    Q = qr_cp(Y)
    assert Q.shape == (50, 3)
    assert np.linalg.norm(Q.T @ Q - np.eye(3)) <= 1e-14
    assert _rel(Q @ (Q.T @ Y), Y) <= 1e-14
    Yf = rng.standard_normal((40, 7))
    Q = qr_cp(Yf)
    assert Q.shape == (40, 7)
    assert qr_cp(np.zeros((10, 4))).shape == (10, 0)


def test_norm2_power_matches_sigma1():
    rng = np.random.default_rng(9)
    D = rng.standard_normal((120, 80))
    _, s, _ = jacobi_svd(D)
    assert abs(norm2_power(D) - s[0]) <= 1e-11 * s[0]
