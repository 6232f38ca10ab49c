"""CTA-pair pass (tc_pass3.cuh) against the fp64 product: accuracy on ragged
shapes, then c5-shape timing of each route. impl 2 = exact (3 terms), 3 =
with the tf32-rounded small operand (2 terms)."""
import sys

import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402


def rna_tf32(x):
    i = x.contiguous().view(torch.int32)
    return ((i + 0x1000) & ~0x1FFF).view(torch.float32)


def check(m, n, l, kind, impls):
    g = torch.Generator(device="cuda").manual_seed(m + n + l + kind)
    ldm = (m + 3) // 4 * 4
    A = torch.randn((n, ldm), device="cuda", generator=g)[:, :m].t()
    A[::7] *= 1e3
    B = torch.randn(((n if kind == 0 else m), l), device="cuda", generator=g).t().contiguous().t()
    h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
    res = []
    for impl in impls:
        Bref = rna_tf32(B.t()).t() if impl == 3 else B
        ref = (A.double() @ Bref.double()) if kind == 0 else (A.double().t() @ Bref.double())
        out = h.debug_pass(kind, impl, A, B)
        torch.cuda.synchronize()
        e = float(torch.linalg.norm(out.double() - ref) / torch.linalg.norm(ref))
        bound = (A.double().abs() @ Bref.double().abs()) if kind == 0 else (A.double().abs().t() @ Bref.double().abs())
        emax = float(((out.double() - ref).abs() / bound.clamp_min(1e-300)).max())
        det = torch.equal(out, h.debug_pass(kind, impl, A, B))
        res.append("impl %d frob %.2e max %.2e det %d" % (impl, e, emax, det))
    print("m %d n %d l %d kind %d: %s" % (m, n, l, kind, " | ".join(res)), flush=True)


def timing(impls, reps=10):
    m, n, l = 65536, 8192, 120
    A = torch.randn((n, m), device="cuda").t()
    X = torch.randn((l, n), device="cuda").t()
    Q = torch.randn((l, m), device="cuda").t()
    h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
    for kind, B in ((0, X), (1, Q)):
        for impl in impls:
            ms = h.debug_pass_timed(kind, impl, A, B, reps)
            print("c5 kind %d impl %d  %.3f ms  %.0f GB/s (A bytes)" % (kind, impl, ms, m * n * 4 / ms / 1e6),
                  flush=True)


if __name__ == "__main__":
    impls = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3").split(",")]
    for (m, n, l) in [(1036, 612, 40), (512, 1024, 64), (2048, 2056, 120), (4100, 260, 128), (130, 70000, 120),
                      (40000, 300, 120), (1036, 612, 16)]:
        for kind in (0, 1):
            check(m, n, l, kind, impls)
    if "--time" in sys.argv:
        timing(impls)
