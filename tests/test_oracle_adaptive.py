"""Pins for oracle/adaptive.py: the Eq. (7) adaptive rank prediction state
machine and the Prop. 4 residual singular value estimate
(P:408-438), against hand-written sequences, the Gaussian closed form behind
Lemma 3 and Monte-Carlo coverage."""
import math

import numpy as np

from oracle import rpca_ialm
from oracle.adaptive import ap_bound, ap_initial, ap_next, residual_sigma_estimate, sketch_varsigma


def test_eq7_state_machine_by_hand():
    """b = ceil(0.1 * 120) = 12, l_0 = ceil(1.2) = 2, a = 2, ceil(rho n) = 5.
    Kept ranks 2, 5, 7, 7, 9, 9, 12, 3 give, by Eq. (7):
      r=2 == l=2  -> p=5, l=min(7, 12)=7
      r=5 <  7    -> p=2, l=7
      r=7 == 7    -> p=5, l=12
      r=7 <  12   -> p=2, l=9
      r=9 == 9    -> p=5, l=12
      r=9 <  12   -> p=2, l=11
      r=12 > 11?  (a kept rank above the width cannot occur; r=11 == 11) -> p=5, l=12
      r=3 <  12   -> p=2, l=5"""
    b = ap_bound(120, 0.1)
    assert b == 12
    l = ap_initial(b)
    assert l == 2
    seq = []
    for r in (2, 5, 7, 7, 9, 9, 11, 3):
        p, l = ap_next(r, l, 2, 5, b)
        seq.append((p, l))
    assert seq == [(5, 7), (2, 7), (5, 12), (2, 9), (5, 12), (2, 11), (5, 12), (2, 5)]


def test_lemma3_constant_on_rank_one():
    """A = s u v^T: ||A w|| = s |v^T w| with v^T w ~ N(0, 1), so the estimate
    alpha sqrt(2/pi) s |g| has mean alpha (2/pi) s and falls below s = sigma_1
    exactly when |g| < 1 / (alpha sqrt(2/pi)) (probability 1 - 0.95 at alpha = 20)."""
    rng = np.random.default_rng(3)
    u = rng.standard_normal(30)
    u /= np.linalg.norm(u)
    v = rng.standard_normal(20)
    v /= np.linalg.norm(v)
    s = 3.0
    A = s * np.outer(u, v)
    est = np.array([residual_sigma_estimate(A, None, rng.standard_normal(20), 20.0) for _ in range(20000)])
    assert abs(est.mean() / (20.0 * (2.0 / math.pi) * s) - 1.0) < 0.02
    p_below = float(np.mean(est < s))
    p_exact = math.erf(1.0 / (20.0 * math.sqrt(2.0 / math.pi)) / math.sqrt(2.0))
    assert abs(p_below - p_exact) < 0.006 and p_exact < 0.05


def test_prop4_coverage():
    """Prop. 4: varsigma >= ||(I - QQ^T)A||_2 >= sigma_{k+1}(A) with
    probability >= 1 - 1/alpha = 95% (alpha = 20), for ANY orthonormal Q."""
    rng = np.random.default_rng(11)
    hits_norm, hits_sigma, N = 0, 0, 400
    for t in range(N):
        U = np.linalg.qr(rng.standard_normal((60, 40)))[0]
        V = np.linalg.qr(rng.standard_normal((40, 40)))[0]
        sv = np.logspace(0, -3, 40)
        A = (U * sv) @ V.T
        Q = np.linalg.qr(rng.standard_normal((60, 6)))[0] if t % 2 else U[:, :6] + 1e-2 * rng.standard_normal((60, 6))
        Q = np.linalg.qr(Q)[0]
        est = residual_sigma_estimate(A, Q, rng.standard_normal(40), 20.0)
        res2 = np.linalg.norm(A - Q @ (Q.T @ A), 2)
        hits_norm += est >= res2
        hits_sigma += est >= sv[6]
        assert res2 >= sv[6] * (1 - 1e-12)  # variational characterisation (proof of Prop. 4)
    assert hits_norm / N >= 0.93 and hits_sigma / N >= 0.93


def test_sketch_varsigma_exact_when_rank_le_k():
    """rank(A) = 4 and the sketch's other samples span range(A): the residual
    of the last sample is zero (no more sampling needed)."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((50, 4)) @ rng.standard_normal((4, 30))
    assert sketch_varsigma(A, rng.standard_normal((30, 7))) <= 1e-12 * np.linalg.norm(A)
    # with a carry spanning range(A) and two fresh samples
    Qt = np.linalg.qr(A)[0][:, :4]
    assert sketch_varsigma(A, rng.standard_normal((30, 2)), carry=Qt) <= 1e-12 * np.linalg.norm(A)


def test_rpca_with_ap_follows_eq7():
    """The iALM with AP: l_0 = ceil(0.1 b), every later width from Eq. (7) of
    the recorded kept ranks, never above b, and the planted rank recovered."""
    rng = np.random.default_rng(2)
    L0 = rng.standard_normal((120, 5)) @ rng.standard_normal((5, 80))
    S0 = np.where(rng.random((120, 80)) < 0.05, rng.uniform(-20, 20, (120, 80)), 0.0)
    D = L0 + S0
    ap = dict(a=2, rho_n=4, b=16)
    out = rpca_ialm(D, 30, 16, 1, lambda k: np.random.default_rng(100 + k).standard_normal((80, 16)),
                    rp=True, ap=ap, L0=L0, varsigma_alpha=20.0)
    h = out["hist"]
    assert h["l"][0] == 2
    for k in range(1, 30):
        assert h["l"][k] == ap_next(h["r"][k - 1], h["l"][k - 1], 2, 4, 16)[1]
        assert h["r"][k] <= h["l"][k] <= 16
    assert h["r"][-1] == 5
    assert h["nrmse"][-1] <= 1e-6
    assert len(h["varsigma"]) == 30 and all(v >= 0 for v in h["varsigma"])
