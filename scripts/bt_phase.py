"""Phase timing of the one-CTA FRSVT kernel through the probe library
scripts/probes/libbtprobe.so: the kernel is event-timed back to back while
stopping after phase k = 1..6 and in full; differences are the phase costs.
Also the FP64 FMA rate of one SM and of the whole GPU. Not product code.

    python scripts/bt_phase.py [m n l q f64 [c1]]
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
tag = "randn"
if len(sys.argv) > 6 and sys.argv[6] == "c1":
    from synth import make_config
    _, dd = make_config("c1")
    A = dd["A"].to(dt).cuda().t().contiguous().t()
    tag = "c1 data"
Om = omega(7, 0, n, l).to(dt).cuda().t().contiguous().t()
X = torch.empty(n, m, dtype=dt, device="cuda").t()
r = torch.zeros(1, dtype=torch.int32, device="cuda")
sig = torch.zeros(l, dtype=torch.float64, device="cuda")
sw = torch.zeros(1, dtype=torch.int32, device="cuda")
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
P = ctypes.c_void_p


def run(stop, reps):
    for _ in range(reps):
        rc = lib.bt_probe_run(f64, m, n, l, q, P(A.data_ptr()), ctypes.c_long(m), P(Om.data_ptr()),
                              P(X.data_ptr()), ctypes.c_double(1.0), P(r.data_ptr()), P(sig.data_ptr()),
                              int(stop), P(sw.data_ptr()), P(fl.data_ptr()), P(s))
        assert rc == 0, rc


def timed(stop, reps=200):
    run(stop, 10)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(stop, reps)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


full = timed(0)
print("one-CTA FRSVT %dx%d l=%d q=%d %s (%s): %.2f us per launch (back to back); sweeps %d flags %d r %d"
      % (m, n, l, q, "f64" if f64 else "f32", tag, full, int(sw.item()), int(fl.item()), int(r.item())))
names = ["load A + Omega", "sketch + orth", "power steps", "W + Gram partials", "Jacobi", "W U_B, sigma, shrink",
         "compose X"]
prev = 0.0
for k in range(1, 8):
    t = timed(k) if k < 7 else full
    print("  %-22s %7.2f us  (cumulative %7.2f)" % (names[k - 1], t - prev, t))
    prev = t
out = torch.zeros(1, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for blocks, threads in ((1, 256), (148, 1024), (592, 1024)):
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
# latencies (cycles per dependent step; one CTA)
names = ["DFMA", "FFMA", "SHFL f64", "fast rsqrt f64", "IEEE div f64", "sqrt f64", "__syncthreads", "LDS chase",
         "DADD", "LDS f64 + DFMA", "rsqrt.approx.f64", "rcp.approx.f64", "F2F round trip", "SHFL f32"]
for threads in (32, 256, 1024):
    res = torch.zeros(14, dtype=torch.int64, device="cuda")
    lib.lat_probe(threads, 512, P(out.data_ptr()), P(res.data_ptr()), P(s))
    lib.lat_probe(threads, 512, P(out.data_ptr()), P(res.data_ptr()), P(s))
    torch.cuda.synchronize()
    print("latency, %4d threads: " % threads + ", ".join("%s %.1f" % (nm, v / 512.0) for nm, v in zip(names, res.tolist())))
