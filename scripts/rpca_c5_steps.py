"""A few c5 iALM steps (for ncu captures of the per-iteration kernels)."""
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P
from synth import make_config
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg, d = make_config("c5", device="cuda")
D = d["D"]; del d
torch.cuda.empty_cache()
m, n = D.shape
h = P.Frsvt(m, n, cfg.l, cfg.q, rp=True, dtype=torch.float32, seed=cfg.seed)
E = torch.empty_like(D); A = torch.empty_like(D); L = torch.empty_like(D)
st = h.rpca_state(D, E, A, L, norm2_D=444.46)
for k in range(steps):
    r = h.rpca_step(st, finalize=(k == steps - 1), want_resid=True)
print("steps", steps, "resid", r, "r", h.info().r)
