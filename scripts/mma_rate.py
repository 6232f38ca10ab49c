"""Cycles per tcgen05.mma (M = 128) back to back on every SM: tf32 TS, bf16
TS, tf32 SS (N = 128) and tf32 TS N = 256."""
import sys

import torch

sys.path.insert(0, '/root/repo')
import paper_1509_00296_b200 as P  # noqa: E402

m, n, l = 4096, 4096, 120
A = torch.zeros((n, m), device="cuda").t()
B = torch.zeros((l, n), device="cuda").t()
h = P.Frsvt(m, n, l, 1, dtype=torch.float32, seed=1)
for kind, name in enumerate(["tf32 TS N128", "bf16 TS N128", "tf32 SS N128", "tf32 TS N256", "tf32 TS N120"]):
    out = h.debug_pass(0, 140 + kind, A, B)
    out = h.debug_pass(0, 140 + kind, A, B)
    ms = h.debug_pass_timed(0, 140 + kind, A, B, 5)
    print("%-14s %.1f cycles/MMA (CTA 0 clock64), %.3f ms per 8000 MMAs/SM" % (name, float(out[0, 0]), ms))
for kind, name in enumerate(["DFMA", "DMMA m8n8k4"]):
    out = h.debug_pass(0, 150 + kind, A, B)
    out = h.debug_pass(0, 150 + kind, A, B)
    cyc, fl = float(out[0, 0]), float(out[1, 0])
    print("%-12s %.1f fp64 flop/cycle/SM (CTA 0, 512 threads)" % (name, fl / cyc))
