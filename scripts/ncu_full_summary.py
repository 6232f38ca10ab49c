"""One line per kernel launch of an `ncu --set full` report: duration, DRAM
read/write bytes and throughput, tensor-pipe / SM / L2 utilisation, grid,
registers, shared memory.

    python scripts/ncu_full_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "ms"), ("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active", "tens%"),
        ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs"),
        ("launch__shared_mem_per_block_dynamic", "smem")]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True).stdout
    rows = list(csv.reader(io.StringIO(out.decode("utf-8", "replace"))))
    h, units = rows[0], rows[1]
    idx = {k: h.index(k) for k, _ in KEYS if k in h}
    ki = h.index("Kernel Name")
    print("kernel | " + " | ".join(lbl + ("" if k not in idx else " [" + units[idx[k]] + "]") for k, lbl in KEYS))
    for r in rows[2:]:
        vals = [r[idx[k]] if k in idx else "-" for k, _ in KEYS]
        print(r[ki][:60] + " | " + " | ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
