"""Per-kernel device times of one bench step of a config under the torch
profiler (CUPTI activity records, no replay), after warm-up steps.
Usage: python scripts/kprof.py [config] [warm] [--seq]"""
import collections
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
import paper_1509_00296_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c5"
warm = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 2
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
W = bench.Workload(P, name, 1, 0, dev, stream, None)
W.estimate_norm2()
with torch.cuda.stream(stream):
    for _ in range(warm):
        W.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    with torch.cuda.stream(stream):
        W.step()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for ev in prof.events():
    if ev.device_type != torch.autograd.DeviceType.CUDA:
        continue
    t = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    agg[ev.name][0] += 1
    agg[ev.name][1] += t
    seq.append((ev.name, t))
units = W.per_step
tot = sum(v[1] for v in agg.values())
print("%s: %d units per step, device us per unit (sum of kernel times) %.1f, launches per unit %.1f" % (
    name, units, tot / units, len(seq) / units))
for kname, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print("%9.1f us/unit %6.2f%% %6d  %s" % (t / units, 100 * t / tot, c, kname[:110]))
if "--seq" in sys.argv:
    for kname, t in seq[: len(seq) // units * 2]:
        print("   seq %8.1f us  %s" % (t, kname[:100]))
