"""One line per kernel launch of an `ncu --set full` report, every value in
ncu's BASE units (--print-units base: seconds, bytes, percent), converted
here to us and GB: duration, DRAM read/write bytes and throughput,
tensor-pipe / shared-pipe / SM / L2 utilisation, SM clock, grid, registers,
shared memory.

    python scripts/ncu_full_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "rd GB", 1e-9),
        ("dram__bytes_write.sum", "wr GB", 1e-9),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %", 1.0),
        ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor %", 1.0),
        ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tmem %", 1.0),
        ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed", "shared-pipe %", 1.0),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %", 1.0),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2 %", 1.0),
        ("gpc__cycles_elapsed.avg.per_second", "clk GHz", 1e-9),
        ("launch__grid_size", "grid", 1.0), ("launch__registers_per_thread", "regs", 1.0),
        ("launch__shared_mem_per_block_dynamic", "smem KB", 1e-3)]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True).stdout
    rows = list(csv.reader(io.StringIO(out.decode("utf-8", "replace"))))
    h = rows[0]
    idx = {k: h.index(k) for k, _, _ in KEYS if k in h}
    ki = h.index("Kernel Name")
    print("kernel | " + " | ".join(lbl for _, lbl, _ in KEYS))
    print("|".join(["---"] * (len(KEYS) + 1)))
    for r in rows[2:]:
        vals = []
        for k, _, f in KEYS:
            try:
                vals.append("%.4g" % (float(r[idx[k]].replace(",", "")) * f) if k in idx else "-")
            except ValueError:
                vals.append(r[idx[k]])
        print(r[ki][:60] + " | " + " | ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
