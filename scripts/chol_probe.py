"""Phase timing of the CholeskyQR factor kernel on a synthetic Gram (l = 120)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(0)
Y = rng.standard_normal((4000, l)) * np.logspace(0, -4, l)
G = torch.from_numpy(Y.T @ Y)
h = P.Frsvt(4096, 4096, l, 1, dtype=torch.float32, seed=1)
for _ in range(3):
    T, s, st = h.debug_chol(G, stamps=True)
d = np.diff(st.astype(np.float64)) / 1e3
print("s", s, "total us %.1f" % ((st[7] - st[0]) / 1e3))
print("load %.1f | panel0 diag %.1f | panel0 rows %.1f | rest of factorisation %.1f | inverse A %.1f | inverse B %.1f | store %.1f"
      % tuple(d))
Q = Y @ T.double().cpu().numpy()
print("orthogonality of Y T: %.2e" % np.linalg.norm(Q.T @ Q - np.eye(l)))
