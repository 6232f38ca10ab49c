"""BASELINE.json configs c1..c5 as seeded synthetic inputs.

Every matrix is column-major-filled from its own Philox stream:
  1 left factor (G1 / U), 2 right factor (G2 / V), 3 dense noise N,
  4 sparse mask (u < fraction), 5 sparse values (a + (b-a) u, same element
  index), 6 c3 moving-block parameters, 1000+c Omega of call c.
seed_c = SEED0 + c. Factors and L0 are formed in fp64; fp32 configs store
D = fl32(L0 + S0) once and both sides read exactly those values.

Sizes can be overridden (m, n, rank, ...) to build small instances of the same
recipe for parity tests, and (row0, m_local) selects a row shard so each rank
of a multi-GPU run generates only its own rows.
"""
import math
from dataclasses import dataclass, field

import torch

from .philox import normal, normal_at, uniform, uniform_at

SEED0 = 150900296  # arXiv id 1509.00296


@dataclass
class Config:
    name: str
    kind: str            # "svt" | "rpca" | "wsvt"
    dtype: str           # "f64" | "f32"
    m: int
    n: int
    l: int               # sketch width (BASELINE "k")
    q: int               # power iterations (paper eta)
    rp: bool             # range propagation
    iters: int           # ALM iterations / reweighted calls / 1
    params: dict = field(default_factory=dict)

    @property
    def seed(self):
        return SEED0 + int(self.params.get("cfg_index", 0))


CONFIGS = {
    "c1": Config("c1", "svt", "f64", 200, 100, 10, 1, False, 1,
                 dict(cfg_index=1, rank=5, noise=0.01)),
    "c2": Config("c2", "rpca", "f32", 1000, 1000, 60, 1, True, 30,
                 dict(cfg_index=2, rank=50, var=1.0 / 1000, frac=0.10, lo=-50.0, hi=50.0, rho=1.5)),
    "c3": Config("c3", "rpca", "f32", 76800, 200, 10, 2, True, 50,
                 dict(cfg_index=3, rank=3, H=240, W=320, block=16, nblocks=15, rho=1.5)),
    "c4": Config("c4", "wsvt", "f32", 4096, 4096, 120, 2, True, 20,
                 dict(cfg_index=4, rank=100, noise=0.1, C=2.0 * math.sqrt(4096), eps=1e-6)),
    "c5": Config("c5", "rpca", "f32", 65536, 8192, 120, 1, True, 40,
                 dict(cfg_index=5, rank=100, var=1.0 / 65536, frac=0.05, lo=-10.0, hi=10.0, rho=1.5)),
}


def _col_block(gen, seed, stream, rows_total, row0, m_loc, cols, device, chunk=1 << 25):
    """Rows [row0, row0+m_loc) of a rows_total x cols column-major stream
    (element (i, j) is e = i + rows_total*j), generated in column chunks."""
    at = {normal: normal_at, uniform: uniform_at}[gen]
    out = torch.empty((cols, m_loc), dtype=torch.float64, device=device)
    rows = torch.arange(row0, row0 + m_loc, dtype=torch.int64, device=device)
    step = max(1, chunk // max(m_loc, 1))
    for j0 in range(0, cols, step):
        j1 = min(cols, j0 + step)
        cj = torch.arange(j0, j1, dtype=torch.int64, device=device)
        e = rows[None, :] + rows_total * cj[:, None]
        out[j0:j1] = at(seed, stream, e)
    return out.t()


def _normal(seed, stream, rows, cols, device, std=1.0, row0=0, m_loc=None):
    m_loc = rows if m_loc is None else m_loc
    if row0 == 0 and m_loc == rows:
        # one contiguous stream range
        from .philox import normal_matrix
        return normal_matrix(seed, stream, rows, cols, device=device, std=std)
    x = _col_block(normal, seed, stream, rows, row0, m_loc, cols, device)
    return x * std if std != 1.0 else x


def _uniform(seed, stream, rows, cols, device, row0=0, m_loc=None):
    m_loc = rows if m_loc is None else m_loc
    if row0 == 0 and m_loc == rows:
        from .philox import uniform_matrix
        return uniform_matrix(seed, stream, rows, cols, device=device)
    return _col_block(uniform, seed, stream, rows, row0, m_loc, cols, device)


def make_config(name, device="cpu", row0=0, m_local=None, **over):
    """Build the inputs of config `name` (optionally resized via keyword
    overrides m=, n=, l=, q=, iters=, rank=, ...). Returns (cfg, data) where
    data holds torch tensors on `device`:
      svt : A (fp64), L (fp64 ground-truth low-rank part)
      wsvt: A (fp32)
      rpca: D (fp32), L0 (fp64 ground truth, this shard), S0 (fp64)
    """
    base = CONFIGS[name]
    p = dict(base.params)
    fields = dict(m=base.m, n=base.n, l=base.l, q=base.q, rp=base.rp, iters=base.iters)
    for k, v in over.items():
        if k in fields:
            fields[k] = v
        else:
            p[k] = v
    cfg = Config(base.name, base.kind, base.dtype, fields["m"], fields["n"], fields["l"],
                 fields["q"], fields["rp"], fields["iters"], p)
    m, n, seed = cfg.m, cfg.n, cfg.seed
    m_loc = m if m_local is None else m_local
    data = {}
    if name == "c1":
        k = p["rank"]
        G1 = _normal(seed, 1, m, k, device, row0=row0, m_loc=m_loc)
        G2 = _normal(seed, 2, n, k, device)
        N = _normal(seed, 3, m, n, device, std=p["noise"], row0=row0, m_loc=m_loc)
        L = G1 @ G2.t()
        data["L"] = L
        data["A"] = _colmajor(L + N)
    elif name == "c4":
        k = p["rank"]
        G1 = _normal(seed, 1, m, k, device, row0=row0, m_loc=m_loc)
        G2 = _normal(seed, 2, n, k, device)
        N = _normal(seed, 3, m, n, device, std=p["noise"], row0=row0, m_loc=m_loc)
        data["A"] = _colmajor((G1 @ G2.t() + N).float())
    elif name in ("c2", "c5"):
        k = p["rank"]
        std = math.sqrt(p["var"])
        U = _normal(seed, 1, m, k, device, std=std, row0=row0, m_loc=m_loc)
        V = _normal(seed, 2, n, k, device, std=std)
        L0 = U @ V.t()
        mask = _uniform(seed, 4, m, n, device, row0=row0, m_loc=m_loc) < p["frac"]
        vals = p["lo"] + (p["hi"] - p["lo"]) * _uniform(seed, 5, m, n, device, row0=row0, m_loc=m_loc)
        S0 = torch.where(mask, vals, torch.zeros_like(vals))
        del mask, vals
        data["L0"] = L0
        data["S0"] = S0
        data["D"] = _colmajor((L0 + S0).float())
    elif name == "c3":
        H, W, B = p["H"], p["W"], p["block"]
        frames = n
        assert H * W == m, "c3: m must equal H*W"
        nb = p["nblocks"]
        k = p["rank"]
        U = _normal(seed, 1, m, k, device)
        V = _normal(seed, 2, n, k, device)
        Xl = U @ V.t()
        # global affine rescale of U V^T to [0,1] (rank 3 + constant)
        L0 = (Xl - Xl.min()) / (Xl.max() - Xl.min())
        S0 = torch.zeros_like(L0)
        bp = uniform(seed, 6, 4 * nb, device="cpu")
        vals = _uniform(seed, 5, m, n, device)
        my, mx = H - (B - 1), W - (B - 1)
        ar = torch.arange(B)
        for b in range(nb):
            y0 = int(math.floor(float(bp[4 * b]) * my))
            x0 = int(math.floor(float(bp[4 * b + 1]) * mx))
            vy = int(math.floor(5 * float(bp[4 * b + 2]))) - 2
            vx = int(math.floor(5 * float(bp[4 * b + 3]))) - 2
            for f in range(frames):
                y = (y0 + f * vy) % my
                x = (x0 + f * vx) % mx
                pix = ((y + ar)[:, None] * W + (x + ar)[None, :]).reshape(-1).to(device)
                S0[pix, f] = vals[pix, f]
        if row0 != 0 or m_loc != m:
            L0, S0 = L0[row0:row0 + m_loc], S0[row0:row0 + m_loc]
        data["L0"] = L0
        data["S0"] = S0
        data["D"] = _colmajor((L0 + S0).float())
    else:
        raise KeyError(name)
    return cfg, data


def _colmajor(x):
    """Column-major storage (the library's layout): a (rows, cols) view whose
    memory is the transpose of a contiguous (cols, rows) tensor."""
    return x.t().contiguous().t()
