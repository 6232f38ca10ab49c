"""Run each tcgen05 pass a few times at c5 size (for ncu capture)."""
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P
m, n, l = 65536, 8192, 120
A = torch.randn((n, m), device="cuda").t()
X = torch.randn((l, n), device="cuda").t()
Q = torch.randn((l, m), device="cuda").t()
h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
for _ in range(2):
    h.debug_pass(0, 1, A, X)
    h.debug_pass(1, 1, A, Q)
torch.cuda.synchronize()
print("ok")
