"""Adaptive rank prediction (AP, §2.3, Eq. (7)) and the
residual singular value estimate (§3.2, Lemma 3 Eq. (13),
Proposition 4 Eq. (14)). fp64 numpy. TEST INFRASTRUCTURE ONLY.

ap_bound(n, gamma)     b = ceil(gamma n), the maximum sampling rate (m >= n)
ap_initial(b)          l_0 = ceil(0.1 b)
ap_next(r, l, a, rho_n, b)
                       Eq. (7): p_{i+1} = a if r_i < l_i else ceil(rho n);
                       l_{i+1} = min(r_i + p_{i+1}, b)
                       with RP the carried basis has r_i columns and the
                       next call draws p = l_{i+1} - r_i fresh ones
residual_sigma_estimate(A, Q, omega, alpha)
                       Prop. 4: varsigma = alpha sqrt(2/pi) ||(I - Q Q^T) A omega||_2,
                       an upper bound of ||(I - QQ^T) A||_2 >= sigma_{k+1}(A)
                       with probability >= 1 - 1/alpha (alpha = 20: 95%)
sketch_varsigma(A, Omega_cols, carry, alpha)
                       the estimate as a by-product of one FRSVT sketch
                       (P:436): y = A omega of the LAST fresh Gaussian column,
                       Q = an orthonormal basis of [Q~, A Omega_{:, :p-1}]

Pinned (tests/test_oracle_adaptive.py) by the Eq. (7) state machine written
out on hand-built rank sequences, by Lemma 3 / Prop. 4 coverage over seeds
(the estimate bounds sigma_{k+1} in >= 93% of draws at alpha = 20), by the
exact case rank(A) <= k (varsigma = 0), and by the closed form of the
expectation of ||G omega|| for a matrix with one nonzero singular value.
"""
import math

import numpy as np


def ap_bound(n, gamma):
    return int(math.ceil(gamma * n))


def ap_initial(b):
    return int(math.ceil(0.1 * b))


def ap_next(r, l, a, rho_n, b):
    """(p_{i+1}, l_{i+1}) from the kept rank r_i and the width l_i (Eq. 7)."""
    p = a if r < l else rho_n
    return p, min(r + p, b)


def residual_sigma_estimate(A, Q, omega, alpha=20.0):
    A = np.asarray(A, dtype=np.float64)
    y = A @ np.asarray(omega, dtype=np.float64)
    if Q is not None and Q.shape[1] > 0:
        y = y - Q @ (Q.T @ y)
    return alpha * math.sqrt(2.0 / math.pi) * float(np.linalg.norm(y))


def sketch_varsigma(A, Omega_cols, carry=None, alpha=20.0):
    """The estimate from one sketch: fresh samples Y = A Omega_cols (n x p),
    basis of the carry and all but the last sample, residual of the last."""
    A = np.asarray(A, dtype=np.float64)
    Om = np.asarray(Omega_cols, dtype=np.float64)
    Y = A @ Om[:, :-1] if Om.shape[1] > 1 else np.zeros((A.shape[0], 0))
    blocks = [Y]
    if carry is not None and carry.shape[1] > 0:
        blocks.insert(0, np.asarray(carry, dtype=np.float64))
    B = np.hstack(blocks)
    Q = np.linalg.qr(B)[0] if B.shape[1] > 0 else None
    return residual_sigma_estimate(A, Q, Om[:, -1], alpha)
