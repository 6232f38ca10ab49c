"""Dense linear-algebra steps of the oracle (fp64, numpy). TEST INFRASTRUCTURE
ONLY — see oracle/__init__.py.

jacobi_svd  : one-sided Hestenes Jacobi SVD — the exact SVD behind Definition 1
              (BASELINE north_star "exact SVT via one-sided
              Jacobi SVD"). Pinned by closed forms (diag, 2x2, rank-deficient),
              by brute force on 2x2/3x2 (characteristic polynomial) and by
              reconstruction/orthogonality invariants (tests/test_oracle_linalg.py).
polar_newton: Newton iteration for the polar decomposition, Definition 2 and
              P:195 ("Newton based polar decomposition suggested by Higham").
              Pinned by W^T W = I, P = P^T >= 0, W P = C, and P^2 = C^T C.
qr_cp       : QR with column pivoting + rank truncation, the rank reveal of
              P:163/P:177 (the paper calls LAPACK dgeqp3 + orgqr; so does this,
              through scipy). Truncation rule: SPEC S:134 (max(m,n)*eps
              relative to |R_11|), reading R4.
norm2_power : block power method for ||D||_2 (mu_0 = 1.25/||D||_2 of the iALM
              schedule). Pinned against the Jacobi sigma_1 on small D.
"""
import numpy as np
import scipy.linalg

EPS = np.finfo(np.float64).eps


def _complete(U, m):
    """Extend the orthonormal columns of U (m x k) to m x m with Gram-Schmidt
    on the identity (deterministic)."""
    cols = [U[:, j] for j in range(U.shape[1])]
    for e in range(m):
        if len(cols) == m:
            break
        v = np.zeros(m)
        v[e] = 1.0
        for _ in range(2):
            for c in cols:
                v -= (c @ v) * c
        nv = np.linalg.norm(v)
        if nv > 1e-8:
            cols.append(v / nv)
    return np.stack(cols, axis=1)


def jacobi_svd(M, tol=1e-15, max_sweeps=60):
    """One-sided Hestenes Jacobi SVD of M (m x n).

    Returns (U, sigma, V) with k = min(m, n): U (m x k) and V (n x k) with
    orthonormal columns, sigma (k,) sorted descending, M = U diag(sigma) V^T.
    Columns of M (of M^T if m < n) are rotated pairwise, cyclic by rows,
    whenever |a_i^T a_j| > tol * ||a_i|| ||a_j||; singular values are the final
    column norms, V accumulates the rotations.
    """
    M = np.array(M, dtype=np.float64)
    m, n = M.shape
    if m < n:
        U, s, V = jacobi_svd(M.T, tol, max_sweeps)
        return V, s, U
    Wk = M.copy()
    V = np.eye(n)
    for _ in range(max_sweeps):
        rotated = False
        for i in range(n - 1):
            for j in range(i + 1, n):
                a = Wk[:, i]
                b = Wk[:, j]
                alpha = a @ a
                beta = b @ b
                gamma = a @ b
                if gamma == 0.0 or abs(gamma) <= tol * np.sqrt(alpha * beta):
                    continue
                rotated = True
                zeta = (beta - alpha) / (2.0 * gamma)
                t = (1.0 if zeta >= 0 else -1.0) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta))
                c = 1.0 / np.sqrt(1.0 + t * t)
                s = c * t
                ai = a.copy()
                Wk[:, i] = c * ai - s * b
                Wk[:, j] = s * ai + c * b
                vi = V[:, i].copy()
                V[:, i] = c * vi - s * V[:, j]
                V[:, j] = s * vi + c * V[:, j]
        if not rotated:
            break
    sigma = np.sqrt(np.sum(Wk * Wk, axis=0))
    order = np.argsort(-sigma, kind="stable")
    sigma = sigma[order]
    Wk = Wk[:, order]
    V = V[:, order]
    nz = sigma > 0
    U = np.zeros((m, n))
    U[:, nz] = Wk[:, nz] / sigma[nz]
    if not np.all(nz):
        k = int(nz.sum())
        U = _complete(U[:, :k], m)[:, :n]
    return U, sigma, V


def polar_newton(C, tol=1e-14, max_iter=100):
    """Polar decomposition C = W P of a square non-singular C (Definition 2,
    P:187-193) by Higham's scaled Newton iteration
        X_{k+1} = (g_k X_k + X_k^{-T} / g_k) / 2,  g_k = (||X_k^{-1}||_F/||X_k||_F)^{1/2},
    scaling switched off once the iteration is in its quadratic phase
    ("Newton based polar decomposition suggested by Higham ...
    converges at a small number of iterations (typically, seven)").
    Returns (W, P, iterations); P is symmetrised.
    """
    X = np.array(C, dtype=np.float64)
    it = 0
    scale = True
    for it in range(1, max_iter + 1):
        Xinv = np.linalg.inv(X)
        if scale:
            g = np.sqrt(np.linalg.norm(Xinv, "fro") / np.linalg.norm(X, "fro"))
        else:
            g = 1.0
        Xn = 0.5 * (g * X + Xinv.T / g)
        delta = np.linalg.norm(Xn - X, "fro") / np.linalg.norm(Xn, "fro")
        X = Xn
        if delta < 1e-2:
            scale = False
        if delta <= tol:
            break
    W = X
    P = W.T @ C
    P = 0.5 * (P + P.T)
    return W, P, it


def qr_cp(Y, tol=None, ref=None):
    """Orthonormal basis of range(Y) by QR with column pivoting, truncated at
    the revealed rank s ("estimating the rank and dominant bases by QR
    decomposition with Column Pivoting"; P:177 dgeqp3 + orgqr).

    Column j of the pivoted R is kept while |R_jj| > tol * ref, with
    tol = max(m, n) * eps and ref = |R_11| unless given.
    Returns Q (m x s).
    """
    Y = np.asarray(Y, dtype=np.float64)
    m, k = Y.shape
    if k == 0:
        return np.zeros((m, 0))
    Q, R, _ = scipy.linalg.qr(Y, mode="economic", pivoting=True)
    d = np.abs(np.diag(R))
    if tol is None:
        tol = max(m, k) * EPS
    if ref is None:
        ref = d[0] if d.size else 0.0
    if ref == 0.0:
        return np.zeros((m, 0))
    s = int(np.sum(d > tol * ref))
    return Q[:, :s]


def norm2_power(D, block=8, max_iter=1000, rtol=1e-13, seed=0):
    """||D||_2 by block power iteration on D^T D with a Rayleigh-Ritz step
    (largest singular value of D X for the orthonormal block X)."""
    D = np.asarray(D, dtype=np.float64)
    rng = np.random.default_rng(seed)
    X = np.linalg.qr(rng.standard_normal((D.shape[1], block)))[0]
    prev = 0.0
    est = 0.0
    for _ in range(max_iter):
        Y = D @ X
        est = np.sqrt(np.max(np.linalg.eigvalsh(Y.T @ Y)))
        X = np.linalg.qr(D.T @ Y)[0]
        if abs(est - prev) <= rtol * est:
            break
        prev = est
    return float(est)
