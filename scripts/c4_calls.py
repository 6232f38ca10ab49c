"""A few c4 reweighted calls (for ncu captures of the small-matrix chain)."""
import sys
import torch
sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
import paper_1509_00296_b200 as P  # noqa: E402
W = bench.Workload(P, sys.argv[1] if len(sys.argv) > 1 else "c4", 1, 0, torch.device("cuda", 0), torch.cuda.current_stream(), None)
W.estimate_norm2()
W.step()
torch.cuda.synchronize()
print("ok", W.h.info().r)
