import torch, time, sys
sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P
m, n, l = 65536, 8192, 120
A = torch.randn((n, m), device="cuda").t()
X = torch.randn((l, n), device="cuda").t()
Q = torch.randn((l, m), device="cuda").t()
h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
for kind, B in ((0, X), (1, Q)):
    for impl in (1, 0):
        h.debug_pass(kind, impl, A, B)
        torch.cuda.synchronize()
        t = time.perf_counter(); reps = 5
        for _ in range(reps):
            h.debug_pass(kind, impl, A, B)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / reps
        print("kind", kind, "impl", impl, "ms %.3f" % (dt * 1e3), "GB/s %.0f" % (m * n * 4 / dt / 1e9))
