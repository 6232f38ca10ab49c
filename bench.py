"""Benchmark of the FRSVT hot path (arXiv 1509.00296) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5] [--impl ours|reference]

Workloads (BASELINE.json configs[0..4]); the default is c5,
the largest config that fits one GPU and the one the north_star's roofline
and scaling targets are quoted on:
  c1  FRSVT calls/s, fp64 200 x 100, l = 10, q = 1; step = 200 calls
  c2  RPCA-iALM iterations/s, fp32 1000 x 1000, l = 60, q = 1, RP; step = one 30-iteration solve
  c3  RPCA-iALM iterations/s, fp32 76800 x 200, l = 10, q = 2, RP; step = one 50-iteration solve
  c4  weighted-FRSVT calls/s, fp32 4096 x 4096, l = 120, q = 2, RP; step = the 20-call reweighted sequence
  c5  RPCA-iALM iterations/s, fp32 65536 x 8192, l = 120, q = 1, RP; step = one 40-iteration solve
A solve step runs init + all iterations (the last one writing L), so every
step mixes the trajectory's r = 0 and steady phases as a solve does. Each
step is replayed as one CUDA graph (the library allocates nothing and never
synchronises inside a call).

N > 1 (torchrun, one process per GPU; `--gpus N` without torchrun re-launches
itself under torch.distributed.run): the rows of the matrix are sharded over
the ranks (strong scaling: the problem is fixed) and the library all-reduces
the Grams, A^T Q and the residual with NCCL.

Reference arm (--impl reference): the fp64 numpy oracle (oracle/) timed as it
stands on this host's cores over a bounded sample of the same workload; rank
0 alone runs it. Neither oracle/ nor libfrsvt is loaded by the other arm.
"""
import argparse
import json
import math
import os
import socket
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

META = {
    "c1": dict(metric="FRSVT calls/s (fp64 200x100, l=10, q=1) on BASELINE c1", unit="calls/s", per_step=200),
    "c2": dict(metric="RPCA-ALM iterations/s (FRSVT l=60, q=1, RP) on BASELINE c2", unit="iter/s"),
    "c3": dict(metric="RPCA-ALM iterations/s (FRSVT l=10, q=2, RP) on BASELINE c3", unit="iter/s"),
    "c4": dict(metric="weighted-FRSVT calls/s (l=120, q=2, RP, reweighted) on BASELINE c4", unit="calls/s"),
    "c5": dict(metric="RPCA-iALM iterations/s (FRSVT l=120, q=1, RP) on BASELINE c5", unit="iter/s"),
}
PASS_GATE = 0.70  # north_star: each pass over A at >= 70% of HBM at 1 GPU
# FP64 FMA issue rate of one SM, measured on this pool's B200 (scripts/bt_phase.py:
# 63.7 DFMA/clk per CTA from clock64, 148 x 1024 threads 34.8 TFLOP/s;
# profiles/r2_fp64_rate.txt): the ALU roof of a one-CTA call (c1)
DFMA_PER_CLK_SM = 64


def _sm_max_mhz():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p)).get("sm_max_mhz", 1965.0))
    return 1965.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _profile_facts(cfg_name, kind):
    """ncu facts of the dominant kernel class `kind` from the committed
    --set full capture (profiles/traffic.json): DRAM bytes per launch and the
    tensor-pipe utilisation, or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p)).get(cfg_name, {}).get(kind)
    if not d:
        return None, None
    return d.get("bytes_per_launch"), d.get("tensor_pipe_pct")


def _finite(x):
    """the JSON line with every non-finite float (an ncu metric without data)
    as null: strict JSON"""
    if isinstance(x, dict):
        return {k: _finite(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [_finite(v) for v in x]
    if isinstance(x, float) and not math.isfinite(x):
        return None
    return x


def alg_bytes_per_unit(cfg):
    """SURVEY §8(d) algorithmic HBM bytes per unit of work (elem = dtype size):
    FRSVT call (2q+3) m n elem (2q+2 reads of A, 1 write of X); iALM iteration
    (2q+6) m n elem ((2q+1) reads of A with the next sketch fused, plus the
    20 B/elem epilogue)."""
    es = 8 if cfg.dtype == "f64" else 4
    mn = cfg.m * cfg.n
    if cfg.kind == "rpca":
        return es * mn * (2 * cfg.q + 6)
    return es * mn * (2 * cfg.q + 3)


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
        return {"sm_mhz": load[len(load) // 2], "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _relaunch_distributed(args):
    """`--gpus N` (N > 1) outside torchrun: run this script under
    torch.distributed.run with N ranks on this node (rank 0 prints the line)."""
    if args.impl == "ours" and torch.cuda.is_available() and torch.cuda.device_count() < args.gpus:
        print(json.dumps({"error": "--gpus %d but only %d CUDA devices visible" % (args.gpus, torch.cuda.device_count())}))
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def _dist(backend):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        return ws, rank, local, dist
    return 1, 0, local, None


def _config_dict(cfg, ws, name):
    kinds = {"svt": "FRSVT call", "wsvt": "reweighted weighted-FRSVT sequence", "rpca": "RPCA-iALM solve"}
    per = META[name].get("per_step", cfg.iters)
    return {"workload": "%s: %s %dx%d %s, FRSVT l=%d q=%d%s, %d %s per step" % (
        name, kinds[cfg.kind], cfg.m, cfg.n, cfg.dtype, cfg.l, cfg.q, " RP" if cfg.rp else "", per,
        "iterations" if cfg.kind == "rpca" else "calls"),
        "m": cfg.m, "n": cfg.n, "l": cfg.l, "q": cfg.q, "range_propagation": cfg.rp,
        "units_per_step": per, "parallelism": "rows%d" % ws,
        "l2_policy": ("inputs larger than L2 (126 MB)" if cfg.m * cfg.n * 4 > 126e6 else
                      "L2-resident inputs (%.1f MB < 126 MB L2): the BASELINE shape, no flush" % (
                          cfg.m * cfg.n * (8 if cfg.dtype == "f64" else 4) / 1e6))}


# ----------------------------------------------------------------- reference arm
def _oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([t.get("num_threads", 1) for t in threadpool_info()] or [os.cpu_count()])
    except Exception:
        return os.cpu_count()


def oracle_rate(name, budget_s=20.0, ref_rows=None):
    """Time the oracle (fp64 numpy, as it stands) on a bounded sample of the
    workload; returns (units/s at full size, sample description, seconds)."""
    import numpy as np

    import oracle
    from synth import CONFIGS, make_config, omega
    base = CONFIGS[name]
    if name == "c1":
        cfg, d = make_config("c1")
        A = d["A"].numpy()
        tau = 0.5 * np.linalg.svd(d["L"].numpy(), compute_uv=False)[4]
        n_calls, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < min(budget_s, 5.0) or n_calls < 3:
            oracle.frsvt(A, omega(cfg.seed, n_calls, cfg.n, cfg.l).numpy(), cfg.l, cfg.q, tau=tau, rp=False)
            n_calls += 1
        dt = time.perf_counter() - t0
        return n_calls / dt, "full c1, %d oracle FRSVT calls (%.1f s)" % (n_calls, dt), dt
    if name == "c4":
        cfg, d = make_config("c4")
        A = d["A"].double().numpy()
        t0 = time.perf_counter()
        oracle.frsvt(A, omega(cfg.seed, 0, cfg.n, cfg.l).numpy(), cfg.l, cfg.q, C=cfg.params["C"],
                     eps=cfg.params["eps"], rp=True)
        dt = time.perf_counter() - t0
        return 1.0 / dt, "full c4, call 0 of the reweighted sequence (%.1f s)" % dt, dt
    # RPCA configs: one iteration on a row sample (every oracle pass is linear in m)
    rows = ref_rows or {"c2": base.m, "c3": 8192, "c5": 4096}[name]
    rows = min(rows, base.m)
    cfg, d = make_config(name, row0=0, m_local=rows)
    D = d["D"].double().numpy()
    n2 = oracle.norm2_power(D, max_iter=30)
    iters = 2 if name == "c2" else 1
    t0 = time.perf_counter()
    oracle.rpca_ialm(D, iters, cfg.l, cfg.q, lambda k: omega(cfg.seed, k, cfg.n, cfg.l).numpy(), rp=cfg.rp,
                     norm2=n2, rho=cfg.params["rho"])
    dt = time.perf_counter() - t0
    rate = iters / dt * (rows / base.m)
    return rate, "%d of %d rows of %s, %d iALM iteration(s) (%.1f s); full-size rate = sample rate x %d/%d" % (
        rows, base.m, name, iters, dt, rows, base.m), dt


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    from synth import CONFIGS
    cfg = CONFIGS[args.config]
    vals, sample = [], None
    for i in range(args.warmup + args.steps):
        rate, sample, _ = oracle_rate(args.config, ref_rows=args.ref_rows)
        if i >= args.warmup:
            vals.append(rate)
    value = sum(vals) / len(vals)
    per = META[args.config].get("per_step", cfg.iters)
    threads = _oracle_threads()
    return {"metric": META[args.config]["metric"], "value": value, "unit": META[args.config]["unit"], "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per / value * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(cfg, ws, args.config), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": META[args.config]["unit"], "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": META[args.config]["unit"], "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------- our arm
class Workload:
    """One bench step of config `name` on this rank's row shard: inputs in
    HBM, a handle, and step() enqueueing the whole unit sequence."""

    def __init__(self, P, name, ws, rank, dev, stream, nccl_id):
        from paper_1509_00296_b200.sharding import shard
        from synth import CONFIGS, make_config
        self.name = name
        c0 = CONFIGS[name]
        self.row0, self.m_loc = shard(c0.m, ws, rank)
        self.cfg, data = make_config(name, device=dev, row0=self.row0, m_local=self.m_loc)
        cfg = self.cfg
        self.dtype = torch.float64 if cfg.dtype == "f64" else torch.float32
        self.per_step = META[name].get("per_step", cfg.iters)
        n, l = cfg.n, cfg.l
        with torch.cuda.stream(stream):
            self.h = P.Frsvt(self.m_loc, n, l, cfg.q, rp=cfg.rp, dtype=self.dtype, seed=cfg.seed, stream=stream,
                             nranks=ws, rank=rank, m_global=cfg.m, row0=self.row0, nccl_id=nccl_id)
            mk = lambda: torch.empty((n, self.m_loc), dtype=self.dtype, device=dev).t()  # noqa: E731
            if cfg.kind == "rpca":
                self.inp = data["D"]
                self.E, self.A, self.out = mk(), mk(), mk()
            else:
                self.inp = data["A"]
                self.out = mk()
        if name == "c1":
            # tau = 0.5 sigma_5(L) of the planted low-rank part (input preparation, BASELINE c1)
            self.tau = 0.5 * float(torch.linalg.svdvals(data["L"].double())[4])
        del data
        torch.cuda.empty_cache()
        self.rho = cfg.params.get("rho", 1.5)
        self.norm2 = None
        self.P = P

    def estimate_norm2(self):
        """||D||_2 once, by the library's device block-power estimate (init)."""
        if self.cfg.kind == "rpca":
            st = self.h.rpca_state(self.inp, self.E, self.A, self.out, rho=self.rho, norm2_D=0.0)
            self.h.rpca_step(st, finalize=True)
            self.norm2 = 1.25 / self.h.get_mu()

    def step(self, src=None, out=None):
        src = self.inp if src is None else src
        out = self.out if out is None else out
        h, cfg = self.h, self.cfg
        if cfg.kind == "rpca":
            s = h.rpca_state(src, self.E, self.A, out, rho=self.rho, norm2_D=self.norm2)
            for k in range(cfg.iters):
                h.rpca_step(s, finalize=(k == cfg.iters - 1))
        elif cfg.kind == "svt":
            for _ in range(self.per_step):
                h.apply(src, self.tau, X=out)
        else:
            h.reset_carry()
            C, eps = cfg.params["C"], cfg.params["eps"]
            for t in range(cfg.iters):
                h.apply_weighted(src, self.P.W_RECIPROCAL if t == 0 else self.P.W_REWEIGHTED, C=C, eps=eps,
                                 X=out)


def run_ours(args, ws, rank, local, dist):
    import paper_1509_00296_b200 as P
    from paper_1509_00296_b200.sharding import exchange_unique_id

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    nccl_id = exchange_unique_id(dist, rank, P.Frsvt.unique_id) if ws > 1 else None
    stream = torch.cuda.Stream(device=dev)
    W = Workload(P, args.config, ws, rank, dev, stream, nccl_id)
    cfg, h = W.cfg, W.h
    W.estimate_norm2()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            W.step()
    barrier()
    graph = None
    if not args.no_graph:
        try:
            l0 = h.launches
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream, capture_error_mode="relaxed"):
                W.step()
            per_step_launches = h.launches - l0
            with torch.cuda.stream(stream):
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
                    W.step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    if graph is not None:
        # per-pass events of one more step launched eagerly right after the
        # timed replays (same kernels, same inputs)
        h.profile(True)
        with torch.cuda.stream(stream):
            W.step()
        barrier()
        prof = h.profile_read()
        h.profile(False)
        launches = per_step_launches * args.steps
        prof_steps = 1
    else:
        prof = h.profile_read()
        h.profile(False)
        launches = h.launches - launches0
        prof_steps = args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    units = W.per_step * args.steps
    value = units / (ms_max / 1e3)

    # ---- roofline: the dominant kernel class (per-launch averages), the
    # per-pass fractions against the 0.70 gate, the whole-unit fraction ------
    peak, peak_src = _peaks()
    live = {k: v for k, v in prof.items() if v[1] > 0}
    dom = max(live, key=lambda k: live[k][0])
    dms, dn, dbytes = live[dom]
    step_ms = ms_max / args.steps
    bound, unit = "hbm", "GB/s"
    if dom == "single":
        # one CTA runs the whole call: the roof is that SM's FP64 FMA pipe
        # (FLOPs 2 m n l (2q+3) per call, the library's kind-3 count)
        bound, unit = "alu", "GFLOP/s"
        peak = 2.0 * DFMA_PER_CLK_SM * _sm_max_mhz() / 1e3
        peak_src = "one SM's FP64 FMA rate: %d DFMA/clk (measured) x 2 x %.0f MHz" % (DFMA_PER_CLK_SM, _sm_max_mhz())
    achieved = (dbytes / dn) / ((dms / dn) / 1e3) / 1e9
    per_pass = {}
    for k, (pms, pn, pb) in live.items():
        gbs = pb / (pms / 1e3) / 1e9
        per_pass[k] = {"ms_per_step": pms / prof_steps, "launches_per_step": pn / prof_steps,
                       ("gflops" if k == "single" else "gbs"): gbs, "frac": gbs / peak,
                       "share_of_step": (pms / prof_steps) / step_ms}
        if k not in ("compose", "single"):
            per_pass[k]["meets_0p70_gate"] = gbs / peak >= PASS_GATE
    unit_bytes = alg_bytes_per_unit(cfg) * (W.m_loc / cfg.m)
    unit_gbs = unit_bytes * W.per_step / (step_ms / 1e3) / 1e9
    hbm_peak = _peaks()[0]
    traffic, tensor_pct = _profile_facts(args.config, dom)

    # ---- end to end through the public API from pinned host memory -------
    # Every step copies its input host -> device and reads its result back;
    # the copies run on their own streams, double-buffered, so step i's
    # result is read back and step i+1's input uploaded while step i+1 / i
    # computes (the pipeline of a serving loop). The timed region spans the
    # first upload to the last read-back.
    e2e = None
    if not args.no_e2e:
        src_h = torch.empty((cfg.n, W.m_loc), dtype=W.dtype, pin_memory=True).t()
        src_h.copy_(W.inp.cpu())
        out_h = [torch.empty((cfg.n, W.m_loc), dtype=W.dtype, pin_memory=True).t() for _ in range(2)]
        src_d = [torch.empty_like(W.inp) for _ in range(2)]
        outs = [W.out, torch.empty_like(W.out)]
        cp_in, cp_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        k_e2e = max(1, args.steps)
        # one CUDA graph per staging buffer (the public API calls captured, as a
        # serving loop would replay them), when the timed region used graphs
        e2e_graphs = None
        if graph is not None:
            try:
                e2e_graphs = []
                for b in range(2):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
                        W.step(src_d[b], outs[b])
                    e2e_graphs.append(g)
            except Exception as exc:  # noqa: BLE001 - report and run the calls eagerly
                print("bench: e2e graph capture failed (%s); eager calls" % exc, file=sys.stderr)
                e2e_graphs = None
                torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cp_in.wait_stream(stream)
        cp_out.wait_stream(stream)
        with torch.cuda.stream(cp_in):
            src_d[0].copy_(src_h, non_blocking=True)
            ev_in[0].record(cp_in)
        for i in range(k_e2e):
            b = i % 2
            if i + 1 < k_e2e:  # upload the next input once step i - 1 (its buffer's last user) is done
                if i >= 1:
                    cp_in.wait_event(ev_comp[1 - b])
                with torch.cuda.stream(cp_in):
                    src_d[1 - b].copy_(src_h, non_blocking=True)
                    ev_in[1 - b].record(cp_in)
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_out[b])  # step i - 2's result read back before it is overwritten
            with torch.cuda.stream(stream):
                if e2e_graphs is not None:
                    e2e_graphs[b].replay()
                else:
                    W.step(src_d[b], outs[b])
                ev_comp[b].record(stream)
            cp_out.wait_event(ev_comp[b])
            with torch.cuda.stream(cp_out):
                out_h[b].copy_(outs[b], non_blocking=True)
                ev_out[b].record(cp_out)
        stream.wait_stream(cp_out)
        stream.wait_stream(cp_in)
        e1.record(stream)
        barrier()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nb = W.m_loc * cfg.n * (8 if cfg.dtype == "f64" else 4) * ws
        e2e = {"value": W.per_step * k_e2e / (float(te.item()) / 1e3), "unit": META[args.config]["unit"],
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "steps": k_e2e,
               "copies": "pinned host buffers; uploads and read-backs on their own streams, double-buffered "
                         "(overlapping the neighbouring steps' compute)",
               "cuda_graph": e2e_graphs is not None}
        del src_h, out_h, src_d, outs, e2e_graphs

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, sample, _ = oracle_rate(args.config, ref_rows=args.ref_rows)
        cpu = {"value": rate, "unit": META[args.config]["unit"], "cores": _oracle_threads(), "kind": "oracle",
               "sample": sample}

    # c1 only: the same single-CTA call as independent c1-shaped problems, one
    # per CTA across the GPU in one launch (frsvt_batched_apply_f64, Omega of
    # call 0 shared): the throughput of the design when calls do not depend on
    # each other. Reported beside the sequential-call value, not instead of it.
    batched = None
    if args.config == "c1" and rank == 0:
        from synth import omega as _omega
        nb = 4 * torch.cuda.get_device_properties(dev).multi_processor_count
        Ab = torch.empty((nb, cfg.n, cfg.m), dtype=torch.float64, device=dev).transpose(1, 2)
        Ab.copy_(W.inp.unsqueeze(0).expand(nb, -1, -1))
        Omb = _omega(cfg.seed, 0, cfg.n, cfg.l).to(dev)
        Xb = torch.empty((nb, cfg.n, cfg.m), dtype=torch.float64, device=dev).transpose(1, 2)
        with torch.cuda.stream(stream):
            for _ in range(max(args.warmup, 1)):
                P.batched_apply(Ab, Omb, q=cfg.q, tau=W.tau, X=Xb, stream=stream)
        barrier()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kb = max(args.steps, 1)
        b0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(kb):
                P.batched_apply(Ab, Omb, q=cfg.q, tau=W.tau, X=Xb, stream=stream)
        b1.record(stream)
        barrier()
        bms = b0.elapsed_time(b1)
        batched = {"value": nb * kb / (bms / 1e3), "unit": "calls/s", "calls_per_launch": nb, "launches": kb,
                   "ms_per_launch": bms / kb,
                   "what": "independent c1-shaped fp64 calls, one CTA each (frsvt_batched_apply_f64), Omega of call 0 "
                           "shared; inputs resident in HBM"}
        del Ab, Xb

    if rank != 0:
        return None
    kernel_names = {"AX": "tc_pass3_kernel<AX> (A X passes)", "AtQ": "tc_pass3_kernel<ATQ> (A^T Q passes)",
                    "compose": "tc_compose2_kernel / composition (X or the fused iALM epilogue)",
                    "single": "batched_frsvt_kernel (the whole call in one CTA)"}
    return {"metric": META[args.config]["metric"], "value": value, "unit": META[args.config]["unit"],
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": cfg.dtype, "data": "synthetic (seeded Philox recipes of SURVEY §8(d))",
            "config": dict(_config_dict(cfg, ws, args.config), cuda_graph=graph is not None),
            "roofline": {"bound": bound, "kernel": kernel_names.get(dom, dom), "kind": dom, "achieved": achieved,
                         "peak": peak, "unit": unit, "frac": achieved / peak, "traffic": traffic,
                         "tensor_pipe_pct": tensor_pct, "peak_source": peak_src,
                         "per_pass": per_pass, "pass_gate": PASS_GATE,
                         "unit_algorithmic_bytes": unit_bytes, "unit_gbs": unit_gbs, "unit_frac": unit_gbs / hbm_peak,
                         "per_pass_scope": ("one eager step right after the timed graph replays" if graph is not None
                                            else "all timed steps")},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
            **({"batched": batched} if batched is not None else {})}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(META))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=None)
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every kernel from the host instead of replaying a CUDA graph of each step")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch_distributed(args)
    ws, rank, local, dist = _dist("gloo" if args.impl == "reference" else "nccl")
    if args.impl == "reference":
        line = run_reference(args, ws, rank)
    else:
        line = run_ours(args, ws, rank, local, dist)
    if line is not None:
        print(json.dumps(_finite(line), allow_nan=False), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
