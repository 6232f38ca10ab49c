"""Philox4x32-10 counter-based generator (Salmon et al., SC'11) in plain torch
integer ops, so the same code runs on the host (oracle inputs) and on a CUDA
device (bench inputs for the 2 GB configs).

Stream layout ("Generator specification"):
  key     = (seed mod 2^32, seed >> 32)
  counter = (t mod 2^32, t >> 32, stream, 0)
  uniform element e   : t = e,      u = ((x0>>5)*2^26 + (x1>>6)) * 2^-53
  normal  element e   : t = e // 2, u_a from (x0,x1), u_b from (x2,x3),
                        rad = sqrt(-2 ln(1-u_a)),
                        z = rad*cos(2*pi*u_b) (e even) / rad*sin(2*pi*u_b) (e odd)
  Omega of call c     : stream 1000 + c, n x l column-major standard normals
                        ("Sample Gaussian random matrix",
                         P:219 "dense Gaussian random matrices ... entry-wise").

All 32-bit words live in int64 tensors; products are split into 16-bit halves
so no int64 overflow ever happens (bit-exact on CPU and CUDA).
"""
import math
import torch

_MASK = 0xFFFFFFFF
_M0, _M1 = 0xD2511F53, 0xCD9E8D57
_W0, _W1 = 0x9E3779B9, 0xBB67AE85


def _mulhilo(a, b):
    """(hi, lo) 32-bit halves of a*b for int64 tensors a < 2^32 and a python
    constant b < 2^32, without overflowing int64."""
    b_lo, b_hi = b & 0xFFFF, b >> 16
    t1 = a * b_lo                      # < 2^48
    t2 = a * b_hi                      # < 2^48
    lo_part = t1 + ((t2 & 0xFFFF) << 16)
    lo = lo_part & _MASK
    hi = ((t2 >> 16) + (lo_part >> 32)) & _MASK
    return hi, lo


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox rounds on int64 tensors holding uint32 words; key words are
    python ints. Returns the four output words."""
    for rnd in range(10):
        if rnd:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        hi0, lo0 = _mulhilo(c0, _M0)
        hi1, lo1 = _mulhilo(c2, _M1)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def _words(seed, stream, t):
    k0, k1 = seed & _MASK, (seed >> 32) & _MASK
    c0 = t & _MASK
    c1 = t >> 32
    c2 = torch.full_like(t, stream & _MASK)
    c3 = torch.zeros_like(t)
    return philox4x32_10(c0, c1, c2, c3, k0, k1)


def _u53(x0, x1):
    return ((x0 >> 5).double() * 67108864.0 + (x1 >> 6).double()) * (2.0 ** -53)


def uniform_at(seed, stream, e):
    """fp64 uniforms at arbitrary element indices e (int64 tensor)."""
    x0, x1, _, _ = _words(seed, stream, e)
    return _u53(x0, x1)


def normal_at(seed, stream, e):
    """fp64 standard normals at arbitrary element indices e (int64 tensor)."""
    x0, x1, x2, x3 = _words(seed, stream, e >> 1)
    ua = _u53(x0, x1)
    ub = _u53(x2, x3)
    rad = torch.sqrt(-2.0 * torch.log1p(-ua))
    ang = (2.0 * math.pi) * ub
    return torch.where((e & 1) == 0, rad * torch.cos(ang), rad * torch.sin(ang))


def uniform(seed, stream, count, device="cpu", start=0):
    """fp64 uniforms in [0,1) for elements start..start+count-1 of a stream."""
    t = torch.arange(start, start + count, dtype=torch.int64, device=device)
    x0, x1, _, _ = _words(seed, stream, t)
    return _u53(x0, x1)


def normal(seed, stream, count, device="cpu", start=0):
    """fp64 standard normals for elements start..start+count-1 of a stream
    (Box-Muller on one Philox block per element pair)."""
    e = torch.arange(start, start + count, dtype=torch.int64, device=device)
    x0, x1, x2, x3 = _words(seed, stream, e >> 1)
    ua = _u53(x0, x1)
    ub = _u53(x2, x3)
    rad = torch.sqrt(-2.0 * torch.log1p(-ua))
    ang = (2.0 * math.pi) * ub
    return torch.where((e & 1) == 0, rad * torch.cos(ang), rad * torch.sin(ang))


def normal_matrix(seed, stream, rows, cols, device="cpu", std=1.0, chunk=1 << 26):
    """rows x cols fp64 matrix, column-major fill (element (i,j) is e=i+rows*j),
    returned as a torch tensor with shape (rows, cols). Generated in chunks so
    the 2 GB configs fit in memory."""
    total = rows * cols
    out = torch.empty(total, dtype=torch.float64, device=device)
    for s in range(0, total, chunk):
        c = min(chunk, total - s)
        out[s:s + c] = normal(seed, stream, c, device=device, start=s)
    if std != 1.0:
        out.mul_(std)
    return out.view(cols, rows).t()


def uniform_matrix(seed, stream, rows, cols, device="cpu", chunk=1 << 26):
    total = rows * cols
    out = torch.empty(total, dtype=torch.float64, device=device)
    for s in range(0, total, chunk):
        c = min(chunk, total - s)
        out[s:s + c] = uniform(seed, stream, c, device=device, start=s)
    return out.view(cols, rows).t()


def omega(seed, call, n, l, device="cpu", tf32=False):
    """Omega of FRSVT call `call`: n x l i.i.d. N(0,1), stream 1000+call,
    column-major. tf32=True: the draws as a
    handle with FRSVT_OPT_TF32_OMEGA holds them (fp32, then rounded to tf32:
    round to nearest with ties away, i.e. + 0x1000 and the low 13 mantissa
    bits cleared), returned in fp64 (exactly representable)."""
    om = normal_matrix(seed, 1000 + call, n, l, device=device)
    if not tf32:
        return om
    bits = om.float().contiguous().view(torch.int32).to(torch.int64)
    bits = ((bits + 0x1000) & 0xFFFFE000) & 0xFFFFFFFF
    bits = torch.where(bits >= 1 << 31, bits - (1 << 32), bits).to(torch.int32)
    return bits.view(torch.float32).double().reshape(om.shape)
