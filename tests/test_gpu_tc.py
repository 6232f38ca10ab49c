"""tcgen05 3xTF32 streaming passes (Y = A X, Z = A^T Q) against an fp64
reference of the same product and against the SIMT path, on shapes with
ragged M/K tails (TMA out-of-bounds fill) and every N tile (l = 16..128)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


@pytest.mark.parametrize("m,n,l", [(1036, 612, 4), (76800, 200, 10), (1036, 612, 16), (1036, 612, 37), (512, 1024, 64),
                                   (2048, 2056, 120), (4100, 260, 128), (130, 70000, 120), (40000, 300, 120)])
@pytest.mark.parametrize("kind", [0, 1])
def test_tc_pass_matches_fp64(P, m, n, l, kind):
    g = torch.Generator(device="cuda").manual_seed(m + n + l + kind)
    ldm = (m + 3) // 4 * 4  # TMA needs 16-byte column strides: ld padded to a multiple of 4
    A = torch.randn((n, ldm), device="cuda", generator=g)[:, :m].t()  # column-major m x n, ld ldm
    A[::7] *= 1e3                                                       # wide dynamic range
    B = torch.randn(((n if kind == 0 else m), l), device="cuda", generator=g).t().contiguous().t()
    h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
    ref = (A.double() @ B.double()) if kind == 0 else (A.double().t() @ B.double())
    out_p2 = h.debug_pass(kind, 2, A, B)
    out_si = h.debug_pass(kind, 0, A, B)
    den = torch.linalg.norm(ref)
    e_p2 = float(torch.linalg.norm(out_p2.double() - ref) / den)
    e_si = float(torch.linalg.norm(out_si.double() - ref) / den)
    # fp32-level products: all within a few fp32 ulps of the fp64 product
    assert e_si < 1e-5, e_si  # SIMT accumulates K in fp32 (long K: ~5e-6)
    assert e_p2 < 1e-5, e_p2
    # element-wise: every output within fp32-level error of its |A||B| bound
    # (a wrong tail element cannot hide in the Frobenius ratio)
    bound = (A.double().abs() @ B.double().abs()) if kind == 0 else (A.double().abs().t() @ B.double().abs())
    assert float(((out_p2.double() - ref).abs() / bound.clamp_min(1e-300)).max()) < 2e-5
    # a plain 1xTF32 product would be ~1e-4 off: the split really is in effect
    assert e_p2 < 0.1 * 2.0 ** -11
    # the stream-K pass is deterministic
    assert torch.equal(out_p2, h.debug_pass(kind, 2, A, B))
    # span-only route (impl 3, reading R17): the product of the exact A with
    # the tf32-rounded B, at the same fp32 level
    Bt = (B.t().contiguous().view(torch.int32).add(0x1000).bitwise_and(~0x1FFF)).view(torch.float32).t()
    ref_t = (A.double() @ Bt.double()) if kind == 0 else (A.double().t() @ Bt.double())
    out_t = h.debug_pass(kind, 3, A, B)
    assert float(torch.linalg.norm(out_t.double() - ref_t) / torch.linalg.norm(ref_t)) < 1e-5
    bound_t = (A.double().abs() @ Bt.double().abs()) if kind == 0 else (A.double().abs().t() @ Bt.double().abs())
    assert float(((out_t.double() - ref_t).abs() / bound_t.clamp_min(1e-300)).max()) < 2e-5
