"""Out-of-bounds write checks (compute-sanitizer is closed on this GPU pool):
every operand lives inside a larger buffer whose guard region (rows past m in
each column up to the leading dimension, columns past n) is filled with a
sentinel; after the call the guards must be untouched, read-only inputs
bit-identical, and the results still match the oracle. Covers the one-CTA
path (c1 shape, fp64), the tensor-core path with ragged shapes, the SIMT
route (leading dimension not a multiple of 4), the fused iALM step and a
batched call with gaps between matrices."""
import numpy as np
import pytest
import torch

import oracle
from synth import make_config, omega
from tests.gpu_util import z14

pytestmark = pytest.mark.gpu
SENT = -7.0


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


def guarded(m, n, ld, dtype, fill=None, extra_cols=3):
    """(view m x n column-major with leading dim ld, backing buffer)."""
    buf = torch.full((n + extra_cols, ld), SENT, dtype=dtype, device="cuda")
    v = buf.t()[:m, :n]
    if fill is not None:
        v.copy_(fill)
    return v, buf


def guards_ok(buf, m, n):
    b = buf.t()
    return bool((b[m:, :n] == SENT).all()) and bool((b[:, n:] == SENT).all())


@pytest.mark.parametrize("m,n,l,q,dtype,ldpad", [
    (200, 100, 10, 1, torch.float64, 5),      # one-CTA path (BASELINE c1 shape)
    (1037, 613, 37, 2, torch.float32, 3),     # tensor-core passes, ragged tiles (ld % 4 == 0)
    (1037, 613, 37, 1, torch.float32, 2),     # ld % 4 != 0: SIMT route
    (777, 301, 16, 1, torch.float32, 7),      # l <= 16: narrow applies
])
def test_apply_writes_only_X(P, m, n, l, q, dtype, ldpad):
    rng = np.random.default_rng(m + n)
    A64 = (rng.standard_normal((m, 12)) @ rng.standard_normal((12, n))) + 0.01 * rng.standard_normal((m, n))
    src = torch.from_numpy(A64).to(dtype)
    ld = m + ldpad
    A, abuf = guarded(m, n, ld, dtype, fill=src.cuda())
    X, xbuf = guarded(m, n, ld, dtype)
    a_before = abuf.clone()
    s = np.linalg.svd(src.double().numpy(), compute_uv=False)
    tau = 0.5 * (s[5] + s[6])
    seed = 91 + l
    h = P.Frsvt(m, n, l, q, rp=False, dtype=dtype, seed=seed)
    h.apply(A, tau, X=X)
    torch.cuda.synchronize()
    assert torch.equal(abuf, a_before), "A (read-only) changed"
    assert guards_ok(xbuf, m, n), "write outside X"
    ref = oracle.frsvt(src.double().numpy(), omega(seed, 0, n, l).numpy(), l, q, tau=tau, rp=False)
    assert z14(X, ref.X, src.double().numpy()) <= (1e-4 if dtype == torch.float32 else 1e-10)


def test_rpca_step_writes_only_its_operands(P):
    cfg, d = make_config("c2", m=520, n=300, rank=10, l=24)
    m, n = 520, 300
    ld = m + 4
    D, dbuf = guarded(m, n, ld, torch.float32, fill=d["D"].cuda())
    E, ebuf = guarded(m, n, ld, torch.float32)
    Aop, abuf = guarded(m, n, ld, torch.float32)
    L, lbuf = guarded(m, n, ld, torch.float32)
    d_before = dbuf.clone()
    D64 = D.double().cpu().numpy()
    n2 = oracle.norm2_power(D64)
    h = P.Frsvt(m, n, cfg.l, cfg.q, rp=True, dtype=torch.float32, seed=cfg.seed)
    st = h.rpca_state(D, E, Aop, L, rho=cfg.params["rho"], norm2_D=n2)
    iters = 18
    for k in range(iters):
        h.rpca_step(st, finalize=(k == iters - 1))
    torch.cuda.synchronize()
    assert torch.equal(dbuf, d_before), "D (read-only) changed"
    for name, buf in (("E", ebuf), ("A", abuf), ("L", lbuf)):
        assert guards_ok(buf, m, n), "write outside " + name
    ref = oracle.rpca_ialm(D64, iters, cfg.l, cfg.q, lambda k: omega(cfg.seed, k, n, cfg.l).numpy(), rp=True,
                           norm2=n2, rho=cfg.params["rho"])
    assert np.linalg.norm(L.double().cpu().numpy() - ref["L"]) <= 1e-4 * max(np.linalg.norm(ref["L"]), 1.0)


def test_batched_writes_only_its_matrices(P):
    B, m, n, l = 6, 37, 29, 8
    rng = np.random.default_rng(5)
    A = rng.standard_normal((B, m, n)).astype(np.float32)
    ld, gap = m + 3, 2  # leading dim past m, and whole columns between matrices
    stride = (n + gap) * ld
    buf_a = torch.full((B * stride + 64,), SENT, dtype=torch.float32, device="cuda")
    buf_x = torch.full((B * stride + 64,), SENT, dtype=torch.float32, device="cuda")
    Av = torch.as_strided(buf_a, (B, m, n), (stride, 1, ld))
    Xv = torch.as_strided(buf_x, (B, m, n), (stride, 1, ld))
    Av.copy_(torch.from_numpy(A).cuda())
    a_before = buf_a.clone()
    Om = omega(17, 0, n, l)
    X, r, _ = P.batched_apply(Av, Om, q=1, tau=1.0, X=Xv)
    torch.cuda.synchronize()
    assert torch.equal(buf_a, a_before), "A (read-only) changed"
    mask = torch.ones_like(buf_x, dtype=torch.bool)
    for b in range(B):
        for j in range(n):
            mask[b * stride + j * ld: b * stride + j * ld + m] = False
    assert bool((buf_x[mask] == SENT).all()), "write outside the X matrices"
    for b in range(B):
        ref = oracle.frsvt(A[b].astype(np.float64), Om.numpy(), l, 1, tau=1.0, rp=False)
        assert z14(Xv[b], ref.X, A[b].astype(np.float64)) <= 1e-4
