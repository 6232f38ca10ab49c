"""Time the small-SVD kernel alone on the Gram of a config's last call
(frsvt_debug_small_svd with reps): ms per solve, sweeps, ms per sweep."""
import sys
import torch
sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
import paper_1509_00296_b200 as P  # noqa: E402
for name in (sys.argv[1:] or ["c4", "c2", "c5"]):
    W = bench.Workload(P, name, 1, 0, torch.device("cuda", 0), torch.cuda.current_stream(), None)
    W.estimate_norm2()
    W.step()
    torch.cuda.synchronize()
    sig, UB, G, sw, ms = W.h.debug_small_svd(0, None, reps=20)
    print("%s l=%d: %.1f us per solve, %d sweeps, %.1f us per sweep" % (name, W.cfg.l, ms * 1e3, sw, ms * 1e3 / max(sw, 1)),
          flush=True)
    del W
    torch.cuda.empty_cache()
