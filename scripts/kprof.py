"""Per-kernel device times of steady-state c5 iALM iterations under the torch
profiler (CUPTI activity records, no replay): iterations 20..29 after 20
warm ones. Usage: python scripts/kprof.py [iters] [warm]"""
import collections
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402
from synth import make_config  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg, d = make_config("c5", device="cuda")
D = d["D"]
del d
torch.cuda.empty_cache()
m, n = D.shape
h = P.Frsvt(m, n, cfg.l, cfg.q, rp=True, dtype=torch.float32, seed=cfg.seed)
E = torch.empty_like(D)
A = torch.empty_like(D)
L = torch.empty_like(D)
st = h.rpca_state(D, E, A, L, norm2_D=447.8)
for k in range(warm):
    h.rpca_step(st)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(iters):
        h.rpca_step(st)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
seq = [(ev.name, ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total)
       for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
if "--seq" in sys.argv:
    n_it = len(seq) // iters
    for name, t in seq[:n_it]:
        print("   seq %8.1f us  %s" % (t, name[:90]))
t0, t1 = None, None
for ev in prof.events():
    if ev.device_type != torch.autograd.DeviceType.CUDA:
        continue
    name = ev.name
    agg[name][0] += 1
    agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
print("r", h.info().r, "per-iteration device us (sum of kernel times) %.1f" % (tot / iters))
for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print("%8.1f us/it %6.2f%% %5d  %s" % (t / iters, 100 * t / tot, c, name[:110]))
