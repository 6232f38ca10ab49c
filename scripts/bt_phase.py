"""Phase timing of the one-CTA FRSVT kernel (clock64 stamps through the probe
library scripts/probes/libbtprobe.so) and the FP64 FMA rate of one SM and
of the whole GPU. Not product code.

    python scripts/bt_phase.py [m n l q f64]
"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import omega  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "scripts", "probes", "libbtprobe.so"))
m, n, l, q, f64 = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (200, 100, 10, 1, 1)))
dt = torch.float64 if f64 else torch.float32
torch.manual_seed(0)
A = torch.randn(n, m, dtype=dt, device="cuda").t()
if len(sys.argv) > 6 and sys.argv[6] == "c1":
    from synth import make_config
    _, dd = make_config("c1")
    A = dd["A"].to(dt).cuda().t().contiguous().t()
Om = omega(7, 0, n, l).to(dt).cuda().t().contiguous().t()
X = torch.empty(n, m, dtype=dt, device="cuda").t()
r = torch.zeros(1, dtype=torch.int32, device="cuda")
sig = torch.zeros(l, dtype=torch.float64, device="cuda")
NL = 40
st = torch.zeros(NL, 8, dtype=torch.int64, device="cuda")
sw = torch.zeros(1, dtype=torch.int32, device="cuda")
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
P = ctypes.c_void_p
# back-to-back launches (the GPU stays busy), stamps of each kept
for it in range(NL):
    rc = lib.bt_probe_run(f64, m, n, l, q, P(A.data_ptr()), ctypes.c_long(m), P(Om.data_ptr()), P(X.data_ptr()),
                          ctypes.c_double(1.0), P(r.data_ptr()), P(sig.data_ptr()), P(st[it].data_ptr()),
                          P(sw.data_ptr()), P(fl.data_ptr()), P(s))
    assert rc == 0, rc
torch.cuda.synchronize()
d = (st[:, 1:] - st[:, :-1]).double().cpu()
acc = d[10:].median(dim=0).values
print("sweeps %d flags %d r %d" % (int(sw.item()), int(fl.item()), int(r.item())))
names = ["load A", "sketch+orth", "power its", "W + Gram", "Jacobi", "sigma/shrink", "compose X"]
tot = float(acc.sum())
print("one-CTA FRSVT %dx%d l=%d q=%d %s: %.0f cycles (%.1f us at 1.965 GHz)" % (m, n, l, q, "f64" if f64 else "f32",
                                                                                tot, tot / 1965.0))
for nm, c in zip(names, acc.tolist()):
    print("  %-14s %8.0f cyc  %5.1f%%" % (nm, c, 100 * c / tot))
# event timing of the launch
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for it in range(200):
    lib.bt_probe_run(f64, m, n, l, q, P(A.data_ptr()), ctypes.c_long(m), P(Om.data_ptr()), P(X.data_ptr()),
                     ctypes.c_double(1.0), P(r.data_ptr()), P(sig.data_ptr()), None, None, None, P(s))
e1.record()
torch.cuda.synchronize()
print("event-timed: %.2f us per launch (back to back)" % (e0.elapsed_time(e1) * 1e3 / 200))
# FP64 FMA rate
out = torch.zeros(1, dtype=torch.float64, device="cuda")
for blocks, threads in ((1, 256), (1, 1024), (148, 1024), (592, 1024)):
    cyc = torch.zeros(blocks, dtype=torch.int64, device="cuda")
    iters = 4096
    lib.dfma_rate(blocks, threads, iters, P(out.data_ptr()), P(cyc.data_ptr()), P(s))
    torch.cuda.synchronize()
    e0.record()
    lib.dfma_rate(blocks, threads, iters, P(out.data_ptr()), P(cyc.data_ptr()), P(s))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    c = float(cyc.double().mean())
    fmas = 8.0 * iters * threads
    print("DFMA %4d x %4d: %.2f DFMA/clk per CTA (clock64), whole launch %.2f TFLOP/s"
          % (blocks, threads, fmas / c, 2 * fmas * blocks / (ms / 1e3) / 1e12))
