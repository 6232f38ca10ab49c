"""Algorithm 1 (FRSVT), step by step, fp64 numpy.
TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

Steps and the passages they follow:
  lines 3-6   no RP:  Omega in R^{n x l} (given), Y = A Omega, Q = QR_CP(Y)
              (rank reveal s = min(l, r) by QR-CP)
  lines 7-11  RP:     Omega_p = first p = l - r columns of Omega (reading Z6),
              Y = A Omega_p, Q_Y = PartialOrthogonalization(Q~, Y) by modified
              Gram-Schmidt, Q = [Q~, Q_Y]  (reading Z19)
  lines 13-15 power iteration eta = q times: Q = QR(A A^T Q) (P:140-142,
              P:181); the first step uses QR-CP to re-check the rank
  line 16     [H, C] = QR(A^T Q)
  line 17     [W, P] = PolarDecomposition(C)        (Newton)
  line 18     [V, D] = EigenDecomposition(P)
  line 19     S_tau(A) = (QV) S_tau(D) (HWV)^T      (Eq. 6)
  line 21     Q~ = QV, restricted to the kept columns (Q~ has r
              columns, r = #{sigma_i > t_i})
Thresholds: t_i = tau (SVT), explicit w_i, or the reciprocal rule
t_i = C/(sigma_i + eps) (weighted SVT, footnote 1 P:48; BASELINE c4).

Pinned (tests/test_oracle_frsvt.py) by: exactness on exactly-low-rank and
diagonal inputs (== exact Jacobi SVT), the Prop. 1 identity
X == svt_exact(Q Q^T A), sigma(X) = max(D - tau, 0) and
interlacing, ||P_Q A - X||_2 <= tau (Lemma 1 / Def. 3), tau = 0 => X = Q Q^T A
(S:289), and the RP edge cases p = 0 and Q~ spanning range(A).
"""
from dataclasses import dataclass

import numpy as np

from .linalg import EPS, polar_newton, qr_cp


@dataclass
class FrsvtResult:
    X: np.ndarray          # m x n thresholded output (None if not requested)
    left: np.ndarray       # QV   (m x s)
    right: np.ndarray      # HWV  (n x s)
    sigma: np.ndarray      # D, singular values of B = Q^T A, descending (s,)
    d: np.ndarray          # shrunk values max(sigma_i - t_i, 0)
    t: np.ndarray          # thresholds used
    r: int                 # #{d_i > 0}
    s: int                 # basis width after rank reveal
    carry: np.ndarray      # Q~ for range propagation (m x r)
    polar_iters: int


def partial_orthogonalization(Qt, Y):
    """Modified Gram-Schmidt of the new samples Y against Q~ and each other
    (P:179), with one re-orthogonalisation pass (reading R6). A column whose
    remaining norm is <= max(m,n)*eps times the largest sample norm is
    dropped (rank reveal of the propagated basis)."""
    m = Y.shape[0]
    basis = [Qt[:, j] for j in range(Qt.shape[1])]
    ref = np.max(np.linalg.norm(Y, axis=0)) if Y.size else 0.0
    tol = max(m, Y.shape[1] + len(basis)) * EPS * ref
    new = []
    for j in range(Y.shape[1]):
        y = Y[:, j].astype(np.float64).copy()
        for _ in range(2):
            for b in basis + new:
                y -= (b @ y) * b
        ny = np.linalg.norm(y)
        if ny > tol and ny > 0:
            new.append(y / ny)
    if not new:
        return np.zeros((m, 0))
    return np.stack(new, axis=1)


def thresholds(sigma, tau=None, w=None, C=None, eps=None):
    if tau is not None:
        return np.full(sigma.shape, float(tau))
    if w is not None:
        t = np.full(sigma.shape, np.inf)
        w = np.asarray(w, dtype=np.float64)
        k = min(len(w), len(sigma))
        t[:k] = w[:k]
        return t
    return C / (sigma + eps)


def frsvt(A, Omega, l, q, tau=None, w=None, C=None, eps=None, carry=None,
          rp=True, want_X=True):
    """FRSVT of A with the given Gaussian test matrix Omega (n x l).

    Exactly one of tau (SVT), w (explicit per-index thresholds) or (C, eps)
    (reciprocal weights C/(sigma_i+eps) of this call's sigma) is used.
    carry: Q~ of the previous call (m x r) when range propagation is on.
    """
    A = np.asarray(A, dtype=np.float64)
    Omega = np.asarray(Omega, dtype=np.float64)
    m, n = A.shape
    # ---- Alg. 1 lines 3-12: initial basis --------------------------------
    if rp and carry is not None and carry.shape[1] > 0:
        r_prev = carry.shape[1]
        p = l - r_prev
        if p > 0:
            Y = A @ Omega[:, :p]
            QY = partial_orthogonalization(carry, Y)
            Q = np.hstack([carry, QY])
        else:
            Q = np.array(carry, dtype=np.float64)
    else:
        Y = A @ Omega[:, :l]
        Q = qr_cp(Y)
    # ---- lines 13-15: power iteration -----------------------------------
    for it in range(q):
        Yp = A @ (A.T @ Q)
        Q = qr_cp(Yp) if it == 0 else np.linalg.qr(Yp)[0]
    s = Q.shape[1]
    if s == 0:
        z = np.zeros(0)
        return FrsvtResult(np.zeros((m, n)) if want_X else None, np.zeros((m, 0)),
                           np.zeros((n, 0)), z, z, z, 0, 0, np.zeros((m, 0)), 0)
    # ---- line 16: [H, C] = QR(A^T Q) ------------------------------------
    Bt = A.T @ Q
    Cs = np.linalg.qr(Bt, mode="r")
    if np.min(np.abs(np.diag(Cs))) <= max(n, s) * EPS * np.max(np.abs(np.diag(Cs))):
        # singular core (S:267 recovery): keep the directions of span(Q) that
        # A actually reaches, i.e. an orthonormal basis of range(B), B = Q^T A
        Q = Q @ qr_cp(Bt.T)
        Bt = A.T @ Q
        s = Q.shape[1]
    H, Cc = np.linalg.qr(Bt)
    # ---- lines 17-18: polar decomposition + eigendecomposition ----------
    W, P, pit = polar_newton(Cc)
    ev, V = np.linalg.eigh(P)
    ev = ev[::-1]
    V = V[:, ::-1]
    # ---- line 19 / Eq. (6) -----------------------------------------------
    t = thresholds(ev, tau=tau, w=w, C=C, eps=eps)
    d = np.maximum(ev - t, 0.0)
    d[~np.isfinite(d)] = 0.0
    left = Q @ V
    right = H @ (W @ V)
    X = (left * d) @ right.T if want_X else None
    keep = d > 0
    return FrsvtResult(X, left, right, ev, d, t, int(keep.sum()), s,
                       left[:, keep].copy(), pit)
