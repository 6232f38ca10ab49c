"""Exact thresholding operators (fp64). TEST INFRASTRUCTURE ONLY.

soft_shrink : S_tau(x) = sgn(x) max(|x| - tau, 0)            (Def. 1)
svt_exact   : S_tau(A) = U_A S_tau(Sigma_A) V_A^T             (Eq. 3)
wsvt_exact  : per-index thresholds t_i on sigma_i sorted descending
              (weighted SVT, footnote 1; partial SVT S:272-280)
proj_2ball  : P_tau(A) = U_A min(Sigma_A, tau) V_A^T          (Def. 3)

Pinned by closed forms, the Moreau split A = S_tau(A) + P_tau(A)
(P:248), the proximal optimality certificate ||A - X*||_2 <= tau and
U_r^T (A - X*) V_r = tau I, and brute-force minimisation of Eq. (2) on tiny
matrices (tests/test_oracle_svt.py).
"""
import numpy as np

from .linalg import jacobi_svd


def soft_shrink(x, tau):
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.maximum(np.abs(x) - tau, 0.0)


def svt_exact(A, tau):
    """Returns (X, sigma, r) with r = #{sigma_i > tau} (strict)."""
    U, s, V = jacobi_svd(A)
    d = np.maximum(s - tau, 0.0)
    X = (U * d) @ V.T
    return X, s, int(np.sum(s > tau))


def wsvt_exact(A, t):
    """X = U diag(max(sigma_i - t_i, 0)) V^T with t_i indexed by the rank
    position of sigma_i (descending). t may be shorter than min(m,n); missing
    thresholds are +inf (those components are removed)."""
    U, s, V = jacobi_svd(A)
    tt = np.full(s.shape, np.inf)
    t = np.asarray(t, dtype=np.float64)
    tt[: min(len(t), len(s))] = t[: len(s)]
    d = np.maximum(s - tt, 0.0)
    d[~np.isfinite(d)] = 0.0
    return (U * d) @ V.T, s, int(np.sum(d > 0))


def proj_2ball(A, tau):
    U, s, V = jacobi_svd(A)
    return (U * np.minimum(s, tau)) @ V.T
