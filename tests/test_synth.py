"""Seeded input generators (synth/): Philox KAT, distribution moments,
determinism and the shard layout every multi-GPU rank relies on."""
import json
import os

import numpy as np
import pytest
import torch

from synth import SEED0, make_config, normal, omega, uniform
from synth.philox import normal_matrix, philox4x32_10

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for v in kat["vectors"]:
        ctr = [torch.tensor([int(x, 16)], dtype=torch.int64) for x in v["ctr"]]
        k0, k1 = (int(x, 16) for x in v["key"])
        out = philox4x32_10(*ctr, k0, k1)
        assert [int(w) for w in out] == [int(x, 16) for x in v["out"]]


def test_uniform_range_and_determinism():
    u = uniform(7, 4, 100000)
    assert float(u.min()) >= 0.0 and float(u.max()) < 1.0
    assert torch.equal(u, uniform(7, 4, 100000))
    assert not torch.equal(u, uniform(7, 5, 100000))
    assert not torch.equal(u, uniform(8, 4, 100000))
    # offset windows are slices of the same stream
    assert torch.equal(uniform(7, 4, 1000, start=500), u[500:1500])
    assert abs(float(u.mean()) - 0.5) < 0.005


def test_normal_moments_500x500():
    """mean within 0.02, variance within 1 +- 0.03 at 500x500."""
    z = normal_matrix(3, 1, 500, 500)
    assert abs(float(z.mean())) <= 0.02
    assert abs(float(z.var()) - 1.0) <= 0.03
    # Box-Muller pairs: even/odd elements come from the same block
    e = normal(3, 1, 10)
    assert torch.equal(e, z.t().reshape(-1)[:10])


def test_omega_layout():
    """Omega(call c) is column-major from stream 1000+c; its first p columns
    are a prefix of the same stream (RP consumes columns 0..p-1)."""
    O = omega(11, 3, 50, 8)
    assert O.shape == (50, 8)
    flat = normal(11, 1003, 400)
    assert torch.equal(O[:, 2], flat[100:150])
    assert torch.equal(omega(11, 3, 50, 4), O[:, :4])


@pytest.mark.parametrize("name,kw", [("c2", dict(m=300, n=120, rank=10)),
                                      ("c5", dict(m=512, n=96, rank=8)),
                                      ("c4", dict(m=256, n=128, rank=10))])
def test_row_shards_match_full(name, kw):
    _, full = make_config(name, **kw)
    key = "D" if "D" in full else "A"
    m = kw["m"]
    parts = []
    for r0, ml in ((0, m // 3), (m // 3, m - m // 3)):
        _, sh = make_config(name, row0=r0, m_local=ml, **kw)
        parts.append(sh[key])
    assert torch.equal(torch.cat(parts, 0), full[key])


def test_c3_shape_and_support():
    cfg, d = make_config("c3", m=48 * 64, n=20, H=48, W=64, nblocks=1)
    assert d["D"].shape == (48 * 64, 20)
    # one 16x16 block per frame, values in [0,1)
    nnz = (d["S0"] != 0).sum(0)
    assert int(nnz.max()) <= 256 and int(nnz.min()) >= 200
    L0 = d["L0"]
    assert float(L0.min()) == 0.0 and float(L0.max()) == 1.0
    # rank(L0) = 3 + constant = 4
    s = np.linalg.svd(L0.numpy(), compute_uv=False)
    assert s[3] > 1e-8 * s[0] and s[4] < 1e-10 * s[0]


def test_recipes_are_column_major_and_typed():
    cfg, d = make_config("c2", m=64, n=40, rank=4)
    assert d["D"].dtype == torch.float32 and d["D"].stride() == (1, 64)
    cfg, d = make_config("c1")
    assert d["A"].dtype == torch.float64 and d["A"].stride() == (1, 200)


def _tf32_rna_reference(x32):
    """nearest tf32 (10 explicit mantissa bits) of an fp32 value, ties away from
    zero, found by comparing the two neighbouring candidates exactly in fp64"""
    import math
    if x32 == 0.0:
        return 0.0
    e = math.frexp(abs(x32))[1]          # |x| in [2^(e-1), 2^e)
    q = 2.0 ** (e - 1 - 10)              # tf32 spacing in that binade
    lo = math.floor(abs(x32) / q) * q
    hi = lo + q
    a = abs(x32)
    r = hi if (a - lo) >= (hi - a) else lo
    return math.copysign(r, x32)


def test_omega_tf32_option_rounding():
    """FRSVT_OPT_TF32_OMEGA draws (synth side): the fp32 draw rounded to the
    nearest tf32 value with ties away (NEXT-4 TF32-exact Omega), checked against
    a brute-force nearest-candidate search; entries exactly tf32."""
    full = omega(SEED0, 3, 97, 7)
    t = omega(SEED0, 3, 97, 7, tf32=True)
    assert t.shape == full.shape and t.dtype == torch.float64
    x32 = full.float()
    assert int((t.float().view(torch.int32) & 0x1FFF).abs().max()) == 0
    ref = torch.tensor([_tf32_rna_reference(float(v)) for v in x32.reshape(-1)], dtype=torch.float64)
    assert torch.equal(t.reshape(-1), ref)
    rel = ((t - x32.double()).abs() / x32.double().abs()).max().item()
    assert rel <= 2.0 ** -11
