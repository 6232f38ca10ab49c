"""Device time of the factor kernels alone (torch profiler): chol_inv (r = 0
and r = 100) vs the blocked orth_chol kernel, l = 120."""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

l = 120
rng = np.random.default_rng(0)
Y = rng.standard_normal((4000, l)) * np.logspace(0, -3, l)
G = torch.from_numpy(Y.T @ Y)
h = P.Frsvt(4096, 4096, l, 1, dtype=torch.float32, seed=1)
for r in (0, 100, 0):
    h.debug_chol_inv(G, r)
h.debug_chol(G)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for r in (0, 100, 60):
        for _ in range(5):
            h.debug_chol_inv(G, r)
    for _ in range(5):
        h.debug_chol(G)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and "kernel" in ev.name:
        print("%8.1f us  %s" % (ev.device_time_total, ev.name[:80]))
for r in (0, 100, 60):
    T, s, st = h.debug_chol_inv(G, r, stamps=True)
    d = np.diff(st[:6].astype(np.float64)) / 1e3
    print("r %3d  load %.1f | schur %.1f | elimination %.1f | T22 %.1f | store %.1f us (%.0f ns per pivot)"
          % ((r,) + tuple(d) + (d[2] * 1e3 / (l - r),)))
