"""Precision probe of the tcgen05 3xTF32 passes vs fp64, as a function of K."""
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P
torch.manual_seed(0)
for (m, n, l) in [(1024, 256, 120), (1024, 2048, 120), (1024, 8192, 120), (65536, 1024, 120)]:
    A = torch.randn((n, m), device="cuda").t()
    X = torch.randn((l, n), device="cuda").t()
    Q = torch.randn((l, m), device="cuda").t()
    h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
    for kind, B in ((0, X), (1, Q)):
        ref = (A.double() @ B.double()) if kind == 0 else (A.double().t() @ B.double())
        den = torch.linalg.norm(ref)
        e = [float(torch.linalg.norm(h.debug_pass(kind, impl, A, B).double() - ref) / den) for impl in (1, 0)]
        # error of a plain fp32 product computed by torch on CUDA cores (no TF32)
        torch.backends.cuda.matmul.allow_tf32 = False
        r32 = (A @ B) if kind == 0 else (A.t() @ B)
        e32 = float(torch.linalg.norm(r32.double() - ref) / den)
        print(f"m={m} n={n} kind={kind} K={n if kind == 0 else m}: tc {e[0]:.2e} simt {e[1]:.2e} torch-fp32 {e32:.2e}")
