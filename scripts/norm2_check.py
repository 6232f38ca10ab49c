"""Device ||D||_2 estimate (library init, reading R7) vs a 200-step fp64 block power method on c5."""
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P
from synth import make_config
cfg, d = make_config("c5", device="cuda")
D = d["D"]; del d
v = torch.randn(cfg.n, 8, device="cuda", dtype=torch.float64)
Dd = D.double()
for it in range(200):
    w = Dd.t() @ (Dd @ v)
    v, _ = torch.linalg.qr(w)
s = torch.linalg.svdvals(Dd @ v)
print("power-method sigma_1..4", s[:4].tolist())
for q in (6,):
    h0 = P.Frsvt(cfg.m, cfg.n, cfg.l, cfg.q, rp=True, dtype=torch.float32, seed=cfg.seed)
    E, A, L = torch.empty_like(D), torch.empty_like(D), torch.empty_like(D)
    st = h0.rpca_state(D, E, A, L, norm2_D=0.0)
    h0.rpca_step(st, finalize=True)
    print("device estimate", 1.25 / h0.get_mu(), "info sigma", h0.info().sigma[:4])
