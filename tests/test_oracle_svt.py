"""Pins for the exact thresholding operators (oracle/svt.py): closed forms
(tests/golden/closed_forms.json), the Moreau split, the proximal
optimality certificate of Eq. (2), and brute-force minimisation on tiny
matrices."""
import json
import os

import numpy as np
import pytest

from oracle import jacobi_svd, proj_2ball, soft_shrink, svt_exact, wsvt_exact

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def test_soft_shrink_examples():
    for x, tau, y in GOLD["soft_shrink"]:
        assert soft_shrink(x, tau) == y


def test_svt_closed_forms():
    for case in GOLD["svt"]:
        X, _, r = svt_exact(np.array(case["A"], float), case["tau"])
        assert np.allclose(X, case["X"], atol=1e-14)
        assert r == case["rank"]
    for case in GOLD["proj_2ball"]:
        assert np.allclose(proj_2ball(np.array(case["A"], float), case["tau"]), case["P"], atol=1e-14)
    for case in GOLD["wsvt"]:
        X, _, _ = wsvt_exact(np.array(case["A"], float), case["t"])
        assert np.allclose(X, case["X"], atol=1e-14)


def test_svt_scaled_rotation():
    """A = 2R (R a rotation), tau = 1 -> X = R."""
    th = 1.1
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    X, _, r = svt_exact(2 * R, 1.0)
    assert np.allclose(X, R, atol=1e-14) and r == 2


@pytest.mark.parametrize("seed,shape", [(0, (12, 8)), (1, (8, 12)), (2, (10, 10))])
def test_moreau_split_and_optimality(seed, shape):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal(shape)
    s_all = np.linalg.svd(A, compute_uv=False)
    tau = 0.5 * (s_all[3] + s_all[4])
    X, s, r = svt_exact(A, tau)
    P = proj_2ball(A, tau)
    # Moreau split A = S_tau(A) + P_tau(A), ||P_tau(A)||_2 = min(sigma_1, tau)
    assert np.linalg.norm(A - X - P) <= 1e-13 * np.linalg.norm(A)
    assert abs(np.linalg.norm(P, 2) - min(s_all[0], tau)) <= 1e-12
    # optimality of Eq. (2): A - X is a subgradient tau*G of tau||X||_*,
    # i.e. ||A - X||_2 <= tau and U_r^T (A - X) V_r = tau I_r
    assert np.linalg.norm(A - X, 2) <= tau * (1 + 1e-12)
    U, sx, V = np.linalg.svd(X)
    Ur, Vr = U[:, :r], V[:r].T
    assert np.linalg.norm(Ur.T @ (A - X) @ Vr - tau * np.eye(r)) <= 1e-12 * tau * r
    # sigma(X) = max(sigma - tau, 0), read by an independent Jacobi run on X
    _, sX, _ = jacobi_svd(X)
    assert np.allclose(sX[:r], s[:r] - tau, rtol=1e-12)
    assert np.all(sX[r:] <= 1e-12 * s[0])


def _objective(Xs, A, tau):
    nuc = np.linalg.svd(Xs, compute_uv=False).sum(-1)
    return tau * nuc + 0.5 * np.sum((Xs - A) ** 2, axis=(-2, -1))


@pytest.mark.parametrize("shape", [(2, 2), (3, 2)])
def test_svt_brute_force_minimiser(shape):
    """Eq. (2) is strongly convex, so X* must beat every perturbation."""
    rng = np.random.default_rng(42)
    A = rng.standard_normal(shape)
    tau = 0.5 * np.linalg.svd(A, compute_uv=False)[0]
    X, _, _ = svt_exact(A, tau)
    f0 = _objective(X[None], A, tau)[0]
    for eps in (1e-3, 1e-6):
        D = rng.standard_normal((10000,) + shape)
        f = _objective(X[None] + eps * D, A, tau)
        assert np.all(f >= f0 - 1e-15)


def test_wsvt_constant_weights_is_svt():
    A = np.random.default_rng(7).standard_normal((9, 6))
    X1, _, _ = svt_exact(A, 0.8)
    X2, _, _ = wsvt_exact(A, np.full(6, 0.8))
    assert np.linalg.norm(X1 - X2) <= 1e-14
