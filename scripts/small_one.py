"""A few FRSVT calls at l = 120 (for ncu captures of the small-matrix kernels)."""
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P
m, n, l = 8192, 2048, 120
torch.manual_seed(0)
A = (torch.randn(n, 100, device="cuda") @ torch.randn(100, m, device="cuda")).t()
A += 0.1 * torch.randn(n, m, device="cuda").t()
h = P.Frsvt(m, n, l, 1, rp=True, dtype=torch.float32, seed=3)
for _ in range(3):
    X, info = h.apply(A, 50.0, info=True)
print("r", info.r, "s", info.s, "sweeps", info.sweeps)
