"""Per-CTA global-timer spans of one stream-K pass (dbg bit 6):
entry, A-producer done, flush done, exit — relative to the earliest entry."""
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

kind, dbg = int(sys.argv[1]), int(sys.argv[2])
m, n, l = 65536, 8192, 120
A = torch.randn((n, m), device="cuda").t()
B = torch.randn((l, n if kind == 0 else m), device="cuda").t()
h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
h.debug_pass(kind, 8 + dbg, A, B)
out = h.debug_pass(kind, 8 + (dbg | 64), A, B)
flat = out.t().contiguous().view(-1).view(torch.int64).cpu().numpy()
G = 148
t = flat[40000:40000 + 4 * G].reshape(G, 4).astype(np.float64)
t -= t[:, 0].min()
print("entry  min %.1f max %.1f us" % (t[:, 0].min() / 1e3, t[:, 0].max() / 1e3))
print("A-prod done min %.1f med %.1f max %.1f us" % (t[:, 1].min() / 1e3, np.median(t[:, 1]) / 1e3, t[:, 1].max() / 1e3))
print("flush done  min %.1f med %.1f max %.1f us" % (t[:, 2].min() / 1e3, np.median(t[:, 2]) / 1e3, t[:, 2].max() / 1e3))
print("exit        min %.1f med %.1f max %.1f us" % (t[:, 3].min() / 1e3, np.median(t[:, 3]) / 1e3, t[:, 3].max() / 1e3))
order = np.argsort(t[:, 2])
print("slowest CTAs (flush done us):", [(int(c), round(t[c, 2] / 1e3, 1)) for c in order[-8:]])
print("fastest CTAs:", [(int(c), round(t[c, 2] / 1e3, 1)) for c in order[:8]])
