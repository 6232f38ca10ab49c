"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
__graft_entry__.smoke() (the single-CTA fp64 call, a tensor-core fp32 call,
a 20-iteration fused iALM solve) plus one batched_apply of 8 small matrices.

    python scripts/sanitize_small.py && \\
    compute-sanitizer --tool memcheck --error-exitcode 99 python scripts/sanitize_small.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.smoke()
import paper_1509_00296_b200 as P  # noqa: E402
from synth import omega  # noqa: E402

rng = np.random.default_rng(3)
A = rng.standard_normal((8, 48, 40)).astype(np.float32)
Ad = torch.from_numpy(np.ascontiguousarray(A.transpose(0, 2, 1))).cuda().transpose(1, 2)
X, r, sig = P.batched_apply(Ad, omega(5, 0, 40, 8), q=1, tau=1.0)
torch.cuda.synchronize()
print("sanitize_small: ok", int(r.sum()))
