"""Benchmark of the FRSVT hot path (arXiv 1509.00296) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Workload (BASELINE.json): config c5 by default — RPCA by inexact ALM on a
65536 x 8192 fp32 matrix (rank-100 Gaussian factors + 5% sparse outliers),
FRSVT with l = 120, q = 1 and range propagation, 40 ALM iterations. It is the
largest config that fits one GPU and the one the north_star's roofline and
scaling targets are quoted on. One bench "step" = one complete 40-iteration
iALM solve (init + 40 rpca_alm_step calls, the last one writing L), so every
step mixes the r = 0 and r = 100 phases of the trajectory exactly as a solve
does. metric = ALM iterations per second of the whole job.

For N > 1 (torchrun, one process per GPU) the rows of D are sharded over the
ranks (strong scaling: the c5 problem is fixed) and the library all-reduces
the Grams, A^T Q and the residual with NCCL.

Reference arm (--impl reference): the fp64 numpy oracle (oracle/) timed as it
stands on this host's cores over a bounded row sample of the same workload.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RPCA-ALM iterations/s (FRSVT l=120, q=1, RP) on BASELINE c5"
UNIT = "iter/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(kernel):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/traffic.json: dram__bytes_read.sum +
    dram__bytes_write.sum), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    e = d.get(kernel)
    return float(e["bytes_per_launch"]) if e else None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", "clocks_%d.csv" % os.getpid())

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": load[len(load) // 2], "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return ws, rank, local, dist
    return 1, 0, local, None


from paper_1509_00296_b200.sharding import exchange_unique_id, shard  # noqa: E402


def _oracle_sample(cfg_name, rows_sample):
    from synth import make_config
    cfg, d = make_config(cfg_name, row0=0, m_local=rows_sample)
    return cfg, d["D"].double().numpy()


def cpu_oracle_rate(cfg, D, iters_sample):
    """Oracle (fp64 numpy, as it stands) on a row sample D of the config's
    matrix: `iters_sample` iALM iterations; returns (full-size iter/s estimate,
    seconds, threads). Every oracle pass is linear in m, so the full-size rate
    is the sample rate times rows_sample/m."""
    import oracle
    from synth import omega
    try:
        from threadpoolctl import threadpool_info
        threads = max([t.get("num_threads", 1) for t in threadpool_info()] or [os.cpu_count()])
    except Exception:
        threads = os.cpu_count()
    n2 = oracle.norm2_power(D, max_iter=30)
    t0 = time.perf_counter()
    oracle.rpca_ialm(D, iters_sample, cfg.l, cfg.q, lambda k: omega(cfg.seed, k, cfg.n, cfg.l).numpy(),
                     rp=cfg.rp, norm2=n2, rho=cfg.params["rho"])
    dt = time.perf_counter() - t0
    rate = iters_sample / dt * (D.shape[0] / cfg.m)
    return rate, dt, threads


def run_reference(args, ws, rank):
    """--impl reference: the oracle is the reference arm (rank 0 only)."""
    if rank != 0:
        return None
    from synth import CONFIGS
    cfg = CONFIGS[args.config]
    rows = args.ref_rows
    cfgs, D = _oracle_sample(args.config, rows)
    times = []
    threads = None
    for i in range(args.warmup + args.steps):
        rate, dt, threads = cpu_oracle_rate(cfgs, D, 1)
        if i >= args.warmup:
            times.append(dt)
    mean_dt = sum(times) / len(times)
    value = (1.0 / mean_dt) * (rows / cfg.m)
    sample = "%d of %d rows of %s, 1 iALM iteration per step (oracle cost is linear in m)" % (
        rows, cfg.m, args.config)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(cfg, ws),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def _config_dict(cfg, ws):
    return {"workload": "%s: RPCA-iALM %dx%d fp32, FRSVT l=%d q=%d RP, %d iterations per step" % (
        cfg.name, cfg.m, cfg.n, cfg.l, cfg.q, cfg.iters),
        "m": cfg.m, "n": cfg.n, "l": cfg.l, "q": cfg.q, "range_propagation": cfg.rp,
        "alm_iters_per_step": cfg.iters, "parallelism": "rows%d" % ws,
        "l2_policy": "inputs larger than L2 (D, E, A are 2.1 GB each; L2 126 MB)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=4096)
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every kernel from the host instead of replaying a CUDA graph of the solve")
    args = ap.parse_args()

    ws, rank, local, dist = _dist()
    if args.impl == "reference":
        line = run_reference(args, ws, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import paper_1509_00296_b200 as P
    from synth import CONFIGS, make_config

    cfg0 = CONFIGS[args.config]
    assert cfg0.kind == "rpca", "bench times the RPCA configs (c2, c3, c5)"
    row0, m_loc = shard(cfg0.m, ws, rank)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg, data = make_config(args.config, device=dev, row0=row0, m_local=m_loc)
    D = data["D"]
    del data
    torch.cuda.empty_cache()
    n, l = cfg.n, cfg.l
    nccl_id = exchange_unique_id(dist, rank, P.Frsvt.unique_id) if ws > 1 else None
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        h = P.Frsvt(m_loc, n, l, cfg.q, rp=cfg.rp, dtype=torch.float32, seed=cfg.seed, stream=stream,
                    nranks=ws, rank=rank, m_global=cfg.m, row0=row0, nccl_id=nccl_id)
        E = torch.empty((n, m_loc), dtype=torch.float32, device=dev).t()
        A = torch.empty_like(E)
        L = torch.empty_like(E)
    rho = cfg.params["rho"]

    # ||D||_2 once (device block-power estimate inside the library's init)
    st = h.rpca_state(D, E, A, L, rho=rho, norm2_D=0.0)
    h.rpca_step(st, finalize=True)
    norm2 = 1.25 / h.get_mu()

    def solve(Dsrc):
        s = h.rpca_state(Dsrc, E, A, L, rho=rho, norm2_D=norm2)
        for k in range(cfg.iters):
            h.rpca_step(s, finalize=(k == cfg.iters - 1))

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        solve(D)
    barrier()
    # The whole 40-iteration solve is one CUDA graph (the library allocates
    # nothing and never synchronises inside rpca_alm_step, and every solve
    # replays the same call sequence from iteration 0); gpu_launches counts
    # the kernels of the captured solve times the replays.
    graph = None
    if not args.no_graph and ws == 1:
        try:
            l0 = h.launches
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream, capture_error_mode="relaxed"):
                solve(D)
            per_solve_launches = h.launches - l0
            with torch.cuda.stream(stream):  # replay() launches on the current stream
                for _ in range(max(1, args.warmup)):
                    graph.replay()
            barrier()
        except Exception as exc:  # noqa: BLE001 - report and time the eager path
            print("bench: CUDA graph capture failed (%s); timing eager launches" % exc, file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    if graph is None:
        launches0 = h.launches
        h.profile(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                if graph is not None:
                    graph.replay()
                else:
                    solve(D)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    if graph is not None:
        # per-kernel events of one more solve, launched eagerly right after the
        # timed replays (same kernels, same inputs, same clocks)
        h.profile(True)
        solve(D)
        barrier()
        prof = h.profile_read()
        h.profile(False)
        launches = per_solve_launches * args.steps
        prof_span = None
    else:
        prof = h.profile_read()
        h.profile(False)
        launches = h.launches - launches0
        prof_span = ms
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = cfg.iters * args.steps / (ms_max / 1e3)

    # ---- roofline of the dominant kernel class (per-launch averages) -----
    peak, peak_src = _peaks()
    dom = max(prof, key=lambda k: prof[k][0])
    dms, dn, dbytes = prof[dom]
    achieved = (dbytes / max(dn, 1)) / ((dms / max(dn, 1)) / 1e3) / 1e9
    per_pass = {k: {"ms_total": v[0], "launches": v[1],
                    "gbs": (v[2] / (v[0] / 1e3) / 1e9) if v[0] > 0 else None,
                    "share_of_step": v[0] / prof_span if prof_span else None} for k, v in prof.items()}

    # ---- end to end through the public API from pinned host memory -------
    e2e = None
    if not args.no_e2e:
        Dh = torch.empty((n, m_loc), dtype=torch.float32, pin_memory=True).t()
        Dh.copy_(D.cpu())
        Lh = torch.empty((n, m_loc), dtype=torch.float32, pin_memory=True).t()
        Dd = torch.empty_like(E)
        k_e2e = max(1, min(args.steps, 3))
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(k_e2e):
                Dd.copy_(Dh, non_blocking=True)
                solve(Dd)
                Lh.copy_(L, non_blocking=True)
        e1.record(stream)
        barrier()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": cfg.iters * k_e2e / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": m_loc * n * 4 * ws, "d2h_bytes_per_step": m_loc * n * 4 * ws,
               "steps": k_e2e}
        del Dh, Lh, Dd

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rows = args.ref_rows
        cfgs, Ds = _oracle_sample(args.config, rows)
        rate, dt, threads = cpu_oracle_rate(cfgs, Ds, 1)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": "%d of %d rows of %s, 1 iALM iteration (%.1f s); full-size rate = sample rate x %d/%d"
                         % (rows, cfg.m, args.config, dt, rows, cfg.m)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(_config_dict(cfg, ws), cuda_graph=graph is not None),
                "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                             "unit": "GB/s", "frac": achieved / peak, "traffic": _traffic(dom),
                             "peak_source": peak_src, "per_pass": per_pass,
                             "per_pass_scope": "one eager solve right after the timed graph replays"
                             if graph is not None else "all timed solves"},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
