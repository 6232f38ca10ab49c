"""Collect a round-end measurement (scripts/gpu_call_final.sh TAG) from
gpurun_out/ into profiles/: bench lines (one JSON per config), per-kernel
profiles, the c5 launch list (compacted) and its per-kernel summary, the ncu
--set full summaries, DRAM bytes per launch of the streaming kernels into
profiles/traffic.json, and a markdown digest profiles/<round>_summary.md.

    python scripts/r2_summary.py TAG [ROUND]      (ROUND defaults to r2)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import launches  # noqa: E402
import ncu_full_summary  # noqa: E402


def last_json(path):
    if not os.path.exists(path):
        return None
    for line in reversed(open(path).read().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


def ncu_rows(rep):
    """rows of an ncu --set full report: from the .ncu-rep, or from the raw
    CSV (base units) written next to it on the GPU box (<stem>_raw.csv)"""
    raw = rep[: -len(".ncu-rep")] + "_raw.csv"
    if os.path.exists(rep):
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                             capture_output=True).stdout.decode("utf-8", "replace")
    elif os.path.exists(raw):
        out = open(raw).read()
    else:
        return []
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        res.append(d)
    return res


def kind_of(name):
    if "tc_compose2_kernel" in name:
        return "compose"
    if "tc_pass3_kernel<0" in name:
        return "AX"
    if "tc_pass3_kernel<1" in name:
        return "AtQ"
    return None


def fnum(d, k):
    try:
        return float(d.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


def main(tag, rnd):
    lines = {}
    for c in ("c1", "c2", "c3", "c4", "c5"):
        j = last_json(os.path.join(OUT, "%s_bench_%s.log" % (tag, c)))
        if j:
            lines[c] = j
            with open(os.path.join(PROF, "%s_bench_%s.json" % (rnd, c)), "w") as f:
                f.write(json.dumps(j) + "\n")
        kp = os.path.join(OUT, "%s_kprof_%s.log" % (tag, c))
        if os.path.exists(kp):
            txt = "\n".join(x for x in open(kp).read().splitlines() if "warn" not in x.lower())
            with open(os.path.join(PROF, "%s_kprof_%s.txt" % (rnd, c)), "w") as f:
                f.write(txt + "\n")
    lc = os.path.join(OUT, "%s_launches.csv" % tag)
    launch_txt = ""
    if os.path.exists(lc):
        subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_compact.py"), lc,
                        os.path.join(PROF, "%s_launches_c5.csv" % rnd)], check=True)
        launch_txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launches.py"), lc],
                                    capture_output=True, text=True).stdout
        with open(os.path.join(PROF, "%s_launch_summary_c5.txt" % rnd), "w") as f:
            f.write(launch_txt)
    # ncu --set full summaries and DRAM bytes per launch of the streaming kernels
    traffic_path = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    ncu_txt = {}
    for c, rep in (("c5", "%s_prof.ncu-rep" % tag), ("c2", "%s_prof_c2.ncu-rep" % tag),
                   ("c3", "%s_prof_c3.ncu-rep" % tag), ("c4", "%s_prof_c4.ncu-rep" % tag)):
        path = os.path.join(OUT, rep)
        summ = path[: -len(".ncu-rep")] + "_summary.txt"
        if os.path.exists(path):
            txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_full_summary.py"), path],
                                 capture_output=True, text=True).stdout
        elif os.path.exists(summ):
            txt = open(summ).read()
        else:
            continue
        ncu_txt[c] = txt
        with open(os.path.join(PROF, "%s_ncu_full_summary_%s.txt" % (rnd, c)), "w") as f:
            f.write(txt)
        best = {}
        for d in ncu_rows(path):
            k = kind_of(d.get("Kernel Name", ""))
            if not k:
                continue
            rd, wr = fnum(d, "dram__bytes_read.sum"), fnum(d, "dram__bytes_write.sum")
            tp = fnum(d, "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
            us = fnum(d, "gpu__time_duration.sum") * 1e-3
            if k not in best or rd + wr > best[k]["bytes_per_launch"]:
                best[k] = {"kernel": d.get("Kernel Name", "")[:80], "bytes_per_launch": rd + wr,
                           "dram_read_bytes": rd, "dram_write_bytes": wr,
                           "tensor_pipe_pct": tp if tp == tp else None,
                           "ncu_us": us,
                           "source": "ncu --set full --clock-control none, gpurun_out/%s (the launch of this kind "
                                     "with the most DRAM bytes: a full pass); profiles/%s_ncu_full_summary_%s.txt"
                                     % (rep, rnd, c)}
        if best:
            traffic.setdefault(c, {}).update(best)
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=2)
    # digest
    md = ["# Round 2 — measurements on one B200 (sm_100a)", "",
          "Collected by `scripts/r2_summary.py %s` from `scripts/gpu_call_final.sh %s` (one gpurun call, one "
          "fresh B200; driver clocks unmodified)." % (tag, tag), "",
          "## Bench lines (`python bench.py --config cN`, defaults: 5 steps, 3 warm-up, CUDA-graph replay)", "",
          "| config | value | unit | ms/step | e2e | oracle (cores) | dominant kernel | roofline frac | per-pass frac | "
          "SM MHz (reasons) |", "|---|---|---|---|---|---|---|---|---|---|"]
    for c in ("c1", "c2", "c3", "c4", "c5"):
        j = lines.get(c)
        if not j:
            md.append("| %s | (missing) |||||||||" % c)
            continue
        rf = j.get("roofline", {})
        pp = rf.get("per_pass", {})
        ppt = ", ".join("%s %.2f" % (k, v.get("frac", 0)) for k, v in pp.items())
        cpu = j.get("cpu_baseline") or {}
        e2e = j.get("e2e") or {}
        clk = j.get("clocks") or {}
        md.append("| %s | %.4g | %s | %.3f | %.4g | %.4g (%s) | %s (%s) | %.3f | %s | %s (%s) |" % (
            c, j["value"], j["unit"], j["ms_per_step"], e2e.get("value", float("nan")),
            cpu.get("value", float("nan")), cpu.get("cores", "-"), rf.get("kind"), rf.get("bound"),
            rf.get("frac", float("nan")), ppt, clk.get("sm_mhz"), ",".join(clk.get("reasons", []))))
    md += ["", "Full JSON lines: `profiles/%s_bench_cN.json`." % rnd, ""]
    for c in ("c5", "c1", "c2", "c3", "c4"):
        kp = os.path.join(PROF, "%s_kprof_%s.txt" % (rnd, c))
        if os.path.exists(kp):
            body = open(kp).read().splitlines()
            md += ["## Per-kernel device time, %s (torch profiler over CUPTI, one bench step after 2 warm-up "
                   "steps; `profiles/%s_kprof_%s.txt`)" % (c, rnd, c), "", "```"] + \
                  [x[:150] for x in body[:12]] + ["```", ""]
    if launch_txt:
        md += ["## ncu launch list of `python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline` (c5)", "",
               "Cold-cache and serialised (`--clock-control none`): compare shares, not absolutes. Compact list: "
               "`profiles/%s_launches_c5.csv`." % rnd, "", "```"] + launch_txt.splitlines()[:20] + ["```", ""]
    for c, txt in ncu_txt.items():
        md += ["## ncu --set full, %s (`profiles/%s_ncu_full_summary_%s.txt`)" % (c, rnd, c), ""] + \
              txt.splitlines()[:18] + [""]
    with open(os.path.join(PROF, "%s_summary.md" % rnd), "w") as f:
        f.write("\n".join(md) + "\n")
    print("wrote", os.path.join(PROF, "%s_summary.md" % rnd))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r2")
