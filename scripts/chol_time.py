"""Time the explicit CholeskyQR factor kernel (chol_inv.cuh) alone through
frsvt_debug_chol_inv (kernel time from CUPTI records, median of 20 calls) and
check Y T orthonormal: python scripts/chol_time.py"""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

for l, r in ((10, 0), (60, 0), (60, 50), (120, 0), (120, 100), (128, 0)):
    h = P.Frsvt(4096, 4096, l, 1, dtype=torch.float32, seed=1)
    rng = np.random.default_rng(l + r)
    m = 3000
    Y = rng.standard_normal((m, l)) * np.logspace(0, -3, l)
    if r:
        Y[:, :r] = np.linalg.qr(rng.standard_normal((m, r)))[0]
    G = torch.from_numpy(Y.T @ Y)
    T, s = h.debug_chol_inv(G, r)
    Tn = T.double().cpu().numpy()
    Q = Y @ Tn[:, :l - r] if r else Y @ Tn
    if r:
        Q = np.concatenate([Y[:, :r], Q], axis=1)
    err = np.linalg.norm(Q.T @ Q - np.eye(l))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(20):
            h.debug_chol_inv(G, r)
        torch.cuda.synchronize()
    ts = sorted(ev.device_time_total for ev in prof.events()
                if ev.device_type == torch.autograd.DeviceType.CUDA and "chol_inv" in ev.name)
    print("l=%3d r=%3d s=%3d |Q^TQ-I|=%.2e  chol_inv median %.1f us (min %.1f, n=%d)" % (
        l, r, s, err, ts[len(ts) // 2], ts[0], len(ts)), flush=True)
    del h
