"""Pins for the Type-B (truncated nuclear norm) iALM with the partial SVT and
the semi-online windows with basis transfer (oracle/rpca.py; PAPER.md P:617,
P:633-645): exactness on an uncorrupted rank-keep input, agreement of the
FRSVT backend with the exact partial SVT backend (S:466-style), and the
windowed driver's stitching and transfer."""
import numpy as np

from oracle import rpca_ialm, wsvt_exact
from oracle.rpca import rpca_windows


def _omf(n, l):
    return lambda k: np.random.default_rng(1000 + k).standard_normal((n, l))


def test_partial_svt_leaves_the_top_values():
    """t = (0, tau, tau, ...): sigma_1 is kept untouched, the others shrunk
    (the PSVT operator the Type-B iALM alternates with)."""
    rng = np.random.default_rng(0)
    U = np.linalg.qr(rng.standard_normal((30, 4)))[0]
    V = np.linalg.qr(rng.standard_normal((20, 4)))[0]
    A = (U * np.array([9.0, 4.0, 2.0, 0.5])) @ V.T
    X, s, r = wsvt_exact(A, np.array([0.0, 1.5, 1.5, 1.5]))
    assert r == 3
    Xe = (U * np.array([9.0, 2.5, 0.5, 0.0])) @ V.T
    assert np.linalg.norm(X - Xe) <= 1e-12 * np.linalg.norm(Xe)


def test_type_b_exact_on_uncorrupted_rank_keep_input():
    """D of rank 1 with no outliers minimises sum_{i>1} sigma_i(L) + lambda||S||_1
    with L = D, S = 0 (objective 0): the iALM with keep = 1 reaches it."""
    rng = np.random.default_rng(1)
    D = np.outer(rng.random(300) + 0.5, rng.random(8) + 0.5)
    out = rpca_ialm(D, 40, 3, 2, _omf(8, 3), keep=1)
    assert np.linalg.norm(out["L"] - D) <= 1e-9 * np.linalg.norm(D)
    assert np.abs(out["E"]).max() <= 1e-9 * np.abs(D).max()


def test_type_b_frsvt_matches_exact_backend():
    rng = np.random.default_rng(2)
    L0 = np.outer(rng.random(200), np.ones(10)) + 0.1 * np.outer(rng.random(200), rng.random(10))
    S0 = np.where(rng.random((200, 10)) < 0.05, rng.random((200, 10)), 0.0)
    D = L0 + S0
    n2 = np.linalg.norm(D, 2)
    ex = rpca_ialm(D, 30, 0, 0, None, backend="exact", keep=1, norm2=n2)
    fr = rpca_ialm(D, 30, 6, 2, _omf(10, 6), keep=1, norm2=n2)
    assert np.linalg.norm(fr["L"] - ex["L"]) <= 1e-6 * np.linalg.norm(ex["L"])


def test_windows_stitch_and_transfer():
    """Stitched windows equal the per-window solves; with a static background
    the transferred and the fresh starts reach the same L."""
    rng = np.random.default_rng(3)
    bg = rng.random(400)
    F = np.outer(bg, np.ones(20))
    D = F + np.where(rng.random((400, 20)) < 0.05, rng.random((400, 20)), 0.0)
    a = rpca_windows(D, 5, 30, 3, 2, _omf(5, 3), keep=1, transfer=True)
    b = rpca_windows(D, 5, 30, 3, 2, _omf(5, 3), keep=1, transfer=False)
    for w in range(4):
        cols = slice(5 * w, 5 * w + 5)
        assert np.array_equal(a["L"][:, cols], a["windows"][w]["L"])
        assert np.linalg.norm(a["L"][:, cols] - b["L"][:, cols]) <= 1e-3 * np.linalg.norm(b["L"][:, cols])
    one = rpca_ialm(np.ascontiguousarray(D[:, :5]), 30, 3, 2, _omf(5, 3), keep=1,
                    norm2=a["windows"][0]["norm2"])
    assert np.array_equal(one["L"], a["windows"][0]["L"])
    # the transferred basis is the previous window's carry
    assert a["windows"][1]["carry"].shape[1] == a["windows"][1]["hist"]["r"][-1]
