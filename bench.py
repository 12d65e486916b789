#!/usr/bin/env python
"""Throughput benchmark of the suite evaluation path (driver contract).

Workload (BASELINE.json metric "function evals/sec at D=100 FP64/FP32";
config 5 on one GPU): one *step* evaluates all 37 functions in float64 and
in float32 on a synthetic population X ~ U[-100,100]^{N x 100}, N = 10^7
(8 GB fp64 + 4 GB fp32, far larger than the 126 MB L2, so every launch
streams X from HBM).  value = 37 * 2 * N * steps / time, whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: one process per GPU.  ``--gpus N`` without a torchrun environment
re-launches itself under ``torch.distributed.run`` with N ranks.  Rows are
sharded (dist.Shard, strong scaling: N fixed); each rank queues its rows'
evaluations without a host synchronisation per call
(Engine.evaluate_async) and the NCCL all-gather of each function's fitness
runs on a communication stream, overlapped with the next function's
evaluation (dist.ShardedEngine.submit); time = max over ranks.

Keys beyond the base contract:
  e2e           same metric through the public API with the population in
                pinned host memory: per step one H2D copy of X, the fp32
                cast, 74 evaluations, one D2H read of every fitness vector.
  roofline      dominant (function, precision) launch: T_roof / T_measured,
                T_roof = max(N*(D+1)*s / HBM, N*F / P_fp),
                F = 2*nnz of the rotations applied; P_fp = measured DMMA fp64
                (fp64) or exact-order FMUL+FADD (fp32) peak on this pool
                (profiles/r02/peaks.json), HBM from MEASURED_PEAKS.json.
  cpu_baseline  the reference's CPU path (the reference package installed in
                baseline/_ref -- else the bit-identical oracle port -- its
                per-point NumPy loop, engine.py:205-209) on min(N, 20000) rows
                on all host cores, plus one pinned core; rank 0, N=1 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "function evals/sec at D=100 FP64/FP32 vs CPU ref; fraction of roofline"
REF_INSTALL = ROOT / "baseline" / "_ref"       # tools/install_reference.sh
UNIT = "evals/s"
PREC = ("double", "single")


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> None:
    """--gpus N > 1 outside torchrun: re-run this command as N ranks (the
    driver's own launch form: torch.distributed.run, 127.0.0.1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), str(Path(__file__).resolve())]
    # the ranks read this command's arguments from the environment (torchrun's
    # own parser would take options such as --n for abbreviations of its own)
    env = dict(os.environ, RB_BENCH_ARGV=json.dumps(sys.argv[1:]))
    sys.exit(subprocess.call(cmd, env=env))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--dim", type=int, default=100)
    ap.add_argument("--rows", "--n", dest="n", type=int, default=10_000_000,
                    help="population rows N (config 5); --rows passes through torchrun unambiguously")
    ap.add_argument("--fns", default="all", help="comma list of ids (default: all 37)")
    ap.add_argument("--precisions", default="double,single")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=20000,
                    help="cpu_baseline: rows in the all-core sample, min(N, this) (BASELINE.md section 2)")
    ap.add_argument("--cpu-rows-1core", type=int, default=400,
                    help="cpu_baseline: rows timed on one pinned core")
    ap.add_argument("--ref-rows", type=int, default=2048,
                    help="--impl reference: rows per step (all cores)")
    ap.add_argument("--breakdown", default="", help="write per-(fn, precision) timings here")
    ap.add_argument("--config", type=int, default=5, choices=(1, 2, 3, 4, 5),
                    help="BASELINE.json config (SURVEY.md 8d): 1 sphere D=10 N=1e3 fp64 (latency); "
                         "2 ids 0-22 D=30 N=1e5; 3 ids 23-28 D=50 N=1e6; 4 ids 29-36 D=100 N=1e6 "
                         "fp64; 5 (default) all 37 D=100 N=1e7")
    ap.add_argument("--e2e-numpy", action="store_true",
                    help="config 5: also time the NumPy host-array path (74 x 8/4 GB H2D per step)")
    argv = json.loads(os.environ["RB_BENCH_ARGV"]) if "RB_BENCH_ARGV" in os.environ else None
    args = ap.parse_args(argv)
    preset = CONFIGS[args.config]
    if args.config != 5:
        args.dim, args.n, args.fns, args.precisions = (preset["dim"], preset["n"], preset["fns"],
                                                       preset["precisions"])
    return args


# BASELINE.json "configs" as SURVEY.md 8d fixes them
CONFIGS = {
    1: {"dim": 10, "n": 1000, "fns": "0", "precisions": "double",
        "name": "shifted-rotated Sphere (f1) D=10, N=1,000 random points, FP64 (latency)"},
    2: {"dim": 30, "n": 100_000, "fns": ",".join(map(str, range(23))), "precisions": "double,single",
        "name": "all basic functions shifted+rotated at D=30, N=100,000, FP64 and FP32"},
    3: {"dim": 50, "n": 1_000_000, "fns": ",".join(map(str, range(23, 29))), "precisions": "double,single",
        "name": "hybrid functions at D=50, N=1,000,000, FP64 and FP32"},
    4: {"dim": 100, "n": 1_000_000, "fns": ",".join(map(str, range(29, 37))), "precisions": "double",
        "name": "composition functions at D=100, N=1,000,000, FP64"},
    5: {"dim": 100, "n": 10_000_000, "fns": "all", "precisions": "double,single",
        "name": "full suite at D=100, N=10^7 (sharded across the GPUs)"},
}


# ----------------------------------------------------------------- helpers
NCU_PIPES = {
    "tensor": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "fma": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "xu": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
}


def ncu_pipes(fn, prec):
    """Pipe utilisation (% of peak while active) of the dominant launch from
    its latest committed ncu --set full summary (profiles/r02/ncu, else
    profiles/r01/v*/), or None:
    the transcendental work the rotate-flop roofline leaves out."""
    import glob
    cands = sorted(glob.glob(str(ROOT / "profiles" / "r01" / "v*" / f"ncu_full_fn{fn}_{prec}.txt")),
                   key=lambda p: int(Path(p).parent.name[1:]))
    cands += glob.glob(str(ROOT / "profiles" / "r02" / "ncu" / f"ncu_full_fn{fn}_{prec}.txt"))
    if not cands:
        return None
    vals = {}
    for line in Path(cands[-1]).read_text().splitlines():
        parts = line.split()
        if len(parts) == 2:
            vals[parts[0]] = parts[1]
    out = {k: round(float(vals[m]), 1) for k, m in NCU_PIPES.items() if m in vals}
    out["source"] = str(Path(cands[-1]).relative_to(ROOT))
    return out


def load_json(path):
    try:
        return json.loads(Path(path).read_text())
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc = index, None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def rotate_flops(pack, fn: int) -> int:
    """F = 2 * nnz of every rotation one evaluation applies."""
    rec = pack.functions[fn]
    total = 0
    for mi in range(rec["member0"], rec["member0"] + rec["n_members"]):
        mem = pack.members[mi]
        for si in range(mem["segment0"], mem["segment0"] + mem["n_segments"]):
            seg = pack.segments[si]
            for gi in range(seg["group0"], seg["group0"] + seg["n_groups"]):
                total += 2 * int(pack.groups[gi]["m"]) ** 2
    return total


# ------------------------------------------------------------ CPU baseline
def _cpu_worker(job):
    dim, fns, precs, rows, core = job
    sys.path.insert(0, str(ROOT))
    if core is not None:
        try:
            os.sched_setaffinity(0, {core})
        except (AttributeError, OSError):
            pass
    if (REF_INSTALL / "robench").exists():
        # the reference itself (tools/install_reference.sh -> baseline/_ref):
        # robench.initialize + Engine.evaluate, its per-point loop
        # (engine.py:205-209); initialize (every evaluator) outside the timing
        sys.path.insert(0, str(REF_INSTALL))
        import robench
        eng = robench.initialize(robench.EngineConfig(dim=dim, max_concurrency=max(rows.shape[0], 1),
                                                      seed=0, threads=1))
        batch = robench.PointBatch(rows)

        def run(fn, p):
            eng.evaluate(fn, batch, p)
    else:
        from oracle.robench_oracle import Oracle
        orc = Oracle(dim, 0)
        for fn in fns:                  # build outside the timed loop (initialize)
            for p in precs:
                orc.evaluator(fn, p)

        def run(fn, p):
            orc.evaluate(fn, rows, p)
    t0 = time.perf_counter()
    n = 0
    for fn in fns:
        for p in precs:
            run(fn, p)
            n += rows.shape[0]
    return n, time.perf_counter() - t0


def cpu_reference(dim, fns, precs, rows_per_proc, x_rows=None, procs=None, n_total=None,
                  pin: bool = False):
    """The reference's per-point path (oracle port, bit-identical to
    robench) on every host core: P processes over disjoint row slices of the
    first rows of the §8d population (pin: process i on core i)."""
    import multiprocessing as mp
    procs = procs or os.cpu_count() or 1
    if x_rows is None:
        from paper_1407_7737_b200.population import host_rows, workload_entropy
        x_rows = host_rows(dim, workload_entropy(dim, n_total or rows_per_proc * procs), 0,
                           rows_per_proc * procs)
    jobs = [(dim, fns, precs, x_rows[i * rows_per_proc:(i + 1) * rows_per_proc], i if pin else None)
            for i in range(procs)]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, jobs)
    evals = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    ref = (REF_INSTALL / "robench").exists()
    return {"value": evals / wall, "unit": UNIT, "cores": procs, "kind": "reference" if ref else "port",
            "sample": (f"{rows_per_proc * procs} rows x {len(fns)} fns x {len(precs)} precisions "
                       f"at D={dim} ({procs} processes x {rows_per_proc} rows, per-point NumPy "
                       f"loop = engine.py:205-209; "
                       + ("the reference package itself, baseline/_ref" if ref else
                          "oracle/robench_oracle.py, the bit-identical port") + ")"),
            "cpu_seconds": sum(r[1] for r in res)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    fns = list(range(37)) if args.fns == "all" else [int(f) for f in args.fns.split(",")]
    precs = [p for p in args.precisions.split(",")]
    procs = os.cpu_count() or 1
    per_proc = max(1, -(-min(args.ref_rows, args.n) // procs))
    for _ in range(max(args.warmup, 0)):
        cpu_reference(args.dim, fns, precs, max(1, per_proc // 8), n_total=args.n)
    vals = [cpu_reference(args.dim, fns, precs, per_proc, n_total=args.n) for _ in range(args.steps)]
    cores = vals[0]["cores"]
    value = statistics.median(v["value"] for v in vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * 37 * len(precs) * args.n / value,
        "ms_per_step_note": ("projected: the full step (every function on all N rows) at the "
                             "sampled rate; each timed step runs the stated row sample"),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64+f32",
        "data": "synthetic X = numpy Philox(SeedSequence((0, D, N, 1001))).uniform(-100, 100), first rows",
        "config": {"workload": f"suite-sweep D={args.dim} N={args.n} (37 fns x {len(precs)} precisions)",
                   "dim": args.dim, "n": args.n, "fns": len(fns), "precisions": precs,
                   "sample": vals[0]["sample"]},
        "cpu_baseline": {k: vals[0][k] for k in ("unit", "cores", "kind", "sample")} | {"value": value},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1407_7737_b200 import EngineConfig, _lib, initialize
    from paper_1407_7737_b200.dist import Shard, ShardedEngine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RB_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0, gloo
    # collectives -- runs the multi-rank code path on a one-GPU box; its
    # numbers are not a scaling measurement
    share = os.environ.get("RB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: --gpus {world} needs {world} GPUs, "
                         f"{torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    D = args.dim
    shard = Shard(rank, world, args.n)
    fns_req = None if args.fns == "all" else [int(f) for f in args.fns.split(",")]
    precs = [p for p in args.precisions.split(",")]
    engine = initialize(EngineConfig(dim=D, max_concurrency=max(shard.count, 1), seed=0,
                                     device=local))
    fns = [f for f in engine.enabled_ids if fns_req is None or f in fns_req]
    flops = {fn: rotate_flops(engine._pack, fn) for fn in fns}

    # the §8d population X = Philox(SeedSequence((0, D, N, 1001))).uniform(-100, 100),
    # drawn on the device bit-identically to numpy; rank r owns its row slice
    from paper_1407_7737_b200.population import uniform_population, workload_entropy
    xs = uniform_population(D, shard.count, workload_entropy(D, args.n), first_row=shard.start,
                            device=local, dtypes=("double", "single"))
    x64, x32 = xs["double"], xs["single"]
    stream = torch.cuda.current_stream()
    sharded = ShardedEngine(engine, shard)
    # inputs smaller than twice the L2 (configs 1-2): calls cycle through
    # copies of X whose total exceeds it, so no call reads a warm X
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    xbytes = shard.count * D * 8
    n_rot = 1 if xbytes >= 2 * l2 else int(min(64, -(-2 * l2 // xbytes)))
    xrot = [xs] + [{p: t.clone() for p, t in xs.items()} for _ in range(n_rot - 1)]
    l2_note = ("inputs larger than L2" if n_rot == 1 else
               f"{n_rot} rotating copies of X ({n_rot * xbytes / 1e6:.0f} MB fp64 > 2 x {l2 / 1e6:.0f} MB L2)")
    dts = {"double": torch.float64, "single": torch.float32}
    # two result slots per precision, reused every other function: the local
    # values and (N > 1 GPUs) the gathered N-vector; slot k % 2 is rewritten
    # only after function k's all-gather has finished (its Pending.done)
    local_bufs = {p: [torch.empty(shard.count, dtype=dts[p], device=dev) for _ in range(2)] for p in precs}
    full_bufs = ({p: [torch.empty(args.n, dtype=dts[p], device=dev) for _ in range(2)] for p in precs}
                 if world > 1 else None)

    per = {}

    def step(record):
        """All functions x precisions queued back to back: no host
        synchronisation per call; statuses checked once at the end."""
        pend = []
        for p in precs:
            for fn in fns:
                k = len(pend)
                if k >= 2:
                    stream.wait_event(pend[k - 2].done)
                if record:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                xk = xrot[(step.calls + k) % n_rot][p]
                pend.append(sharded.submit(fn, xk, p, local_out=local_bufs[p][k % 2],
                                           out=full_bufs[p][k % 2] if full_bufs else None))
                if record:
                    e1.record(stream)
                    per.setdefault((fn, p), []).append((e0, e1, 1))
        for pd in pend:                  # the comm stream's tail joins the step
            stream.wait_event(pd.done)
        step.calls += len(pend)
        return pend

    step.calls = 0

    def check(pend):
        for pd in pend:
            pd.result()

    # world == 1: a step is ONE native call queueing every (function,
    # precision) evaluation (Engine.evaluate_many -> rb_func_evaluate_many),
    # so the device time is not bounded by per-call Python work at small N;
    # N > 1 GPUs: per-call submits, each with its fitness all-gather
    calls = [(fn, p) for p in precs for fn in fns]
    out_bufs = {p: local_bufs[p][0] for p in precs}
    # every call keeps its own values (distinct outputs also let the engine
    # overlap consecutive calls on two streams, rb_func_evaluate_many)
    call_outs = ([torch.empty(shard.count, dtype=dts[p], device=dev) for _, p in calls]
                 if world == 1 else None)

    def step_many():
        k0 = step.calls
        step.calls += len(calls)
        return engine.evaluate_many(calls, [xrot[(k0 + i) % n_rot][p] for i, (fn, p) in enumerate(calls)],
                                    outs=call_outs)

    timed_step = step_many if world == 1 else (lambda: step(False))
    for _ in range(args.warmup):
        check(timed_step())
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    launches0 = _lib.launch_count()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    pends = [timed_step() for _ in range(args.steps)]
    t_end.record(stream)
    torch.cuda.synchronize()
    for pd in pends:
        check(pd)
    barrier()
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    # per-(function, precision) device times (untimed pass): CUDA events
    # around R back-to-back calls of each, queued in one native call (R > 1
    # at small N, where a single launch is shorter than the host work per call)
    reps = 1 if shard.count >= 1_000_000 else 8
    for fn, p in calls:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0 = step.calls
        step.calls += reps
        e0.record(stream)
        pd = engine.evaluate_many([(fn, p)] * reps, [xrot[(k0 + i) % n_rot][p] for i in range(reps)],
                                  outs=[out_bufs[p]] * reps)
        e1.record(stream)
        per[(fn, p)] = [(e0, e1, reps)]
        check(pd)
    torch.cuda.synchronize()
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    evals = args.steps * len(fns) * len(precs) * args.n
    value = evals / (ms / 1e3)

    # per-(fn, precision) device time and roofline
    peaks = load_json(ROOT / "MEASURED_PEAKS.json")
    peaks_file = ROOT / "profiles" / "r02" / "peaks.json"      # tools/peaks_microbench.cu
    mypk = load_json(peaks_file)
    hbm = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
    # compute ceilings of the rotate: DMMA f64 for float64;
    # for float32 the exact-order pair (rounded product + rounded add: two
    # FP32-pipe instructions per MAC, NumPy's rounding rules out FMA/TF32)
    p_fp = {"double": float(mypk.get("dmma_m16n8k4_tflops", 36.9)) * 1e12,
            "single": float(mypk.get("fmul_fadd_tflops", 36.6)) * 1e12}
    rows = []
    for (fn, p), evs in per.items():
        t = sum(a.elapsed_time(b) / r for a, b, r in evs) / 1e3 / len(evs)
        s = 8 if p == "double" else 4
        t_hbm = shard.count * (D + 1) * s / hbm
        t_fp = shard.count * flops[fn] / p_fp[p]
        rows.append({"fn": fn, "precision": p, "seconds": t, "evals_per_s": shard.count / t,
                     "t_roof_hbm": t_hbm, "t_roof_fp": t_fp, "frac": max(t_hbm, t_fp) / t,
                     "rotate_flops_per_eval": flops[fn]})
    rows.sort(key=lambda r: -r["seconds"])
    dom = rows[0]
    bound = "hbm" if dom["t_roof_hbm"] >= dom["t_roof_fp"] else "tensor"
    if bound == "hbm":
        achieved = shard.count * (D + 1) * (8 if dom["precision"] == "double" else 4) / dom["seconds"] / 1e9
        peak, unit = hbm / 1e9, "GB/s"
    else:
        achieved = shard.count * flops[dom["fn"]] / dom["seconds"] / 1e12
        peak, unit = p_fp[dom["precision"]] / 1e12, "TFLOP/s"
    traffic = load_json(ROOT / "profiles" / "r02" / "ncu_traffic.json").get(
        f"{dom['fn']}/{dom['precision']}")
    roofline = {
        "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
        "frac": achieved / peak, "traffic": traffic,
        "kernel": f"rb::evaluate_kernel<{'double' if dom['precision'] == 'double' else 'float'}> "
                  f"fn={dom['fn']}",
        "peak_source": ("MEASURED_PEAKS.json hbm_gbs" if bound == "hbm" else
                        "profiles/r02/peaks.json (tools/peaks_microbench.cu on this pool: "
                        + ("DMMA m16n8k4 f64" if dom["precision"] == "double" else
                           "FMUL+FADD f32 exact-order pair; FFMA peak %s TF/s beside it"
                           % mypk.get("ffma_tflops", "?")) + ")"),
        "suite_frac": sum(max(r["t_roof_hbm"], r["t_roof_fp"]) for r in rows) / sum(r["seconds"] for r in rows),
        # the compute bound is the rotation's 2*nnz flops: DMMA (tensor
        # pipe) in fp64; exact-order SIMT FMUL+FADD in fp32 (NumPy's rounding rules out
        # FMA and TF32 tensor cores); transcendental work is outside F (pipe
        # utilisation in profiles/)
        "compute_pipe": ("fp64 DMMA (mma.sync m16n8k4)" if dom["precision"] == "double"
                         else "fp32 SIMT FMUL+FADD, exact NumPy order"),
        "pipe_utilization": ncu_pipes(dom["fn"], dom["precision"]),
    }

    # e2e through the reference's own call: Engine.evaluate(fn, numpy X,
    # precision) with X in ordinary (pageable) host memory, values back as
    # NumPy -> rb_h_func_evaluate[f], H2D of X and D2H of f in every call
    e2e_numpy = None
    latency = None
    e2e_many = None
    if not args.no_e2e and world == 1 and args.config == 5:
        # the headline e2e: the reference's user holds X as a NumPy array and
        # asks for every (function, precision) -- one C-ABI call with host
        # buffers (Engine.evaluate_many -> rb_h_func_evaluate_many), every
        # host<->device copy inside the timed region
        xh_many = x64.cpu().numpy()
        engine.evaluate_many(calls, xh_many)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            engine.evaluate_many(calls, xh_many)
        wall_m = time.perf_counter() - t0
        e2e_many = {
            "value": args.steps * len(calls) * args.n / wall_m, "unit": UNIT,
            "h2d_bytes_per_step": shard.count * D * 8,
            "d2h_bytes_per_step": sum(shard.count * (8 if p == "double" else 4) for _, p in calls),
            "ms_per_step": 1e3 * wall_m / args.steps,
            "path": ("Engine.evaluate_many([(fn, precision) ...], numpy float64 X) -> "
                     "rb_h_func_evaluate_many (C ABI, host pointers): X staged through pinned "
                     "~128 MB row chunks and uploaded once for all calls, float32 cast on the "
                     "device, every call's values copied back into NumPy arrays"),
            "timing": "host wall clock around the blocking call"}
        del xh_many
    if not args.no_e2e and world == 1 and (args.config != 5 or args.e2e_numpy):
        xh = x64.cpu().numpy()
        call_times = []

        def np_step():
            for p in precs:
                for fn in fns:
                    t0 = time.perf_counter()
                    engine.evaluate(fn, xh, p)
                    call_times.append(time.perf_counter() - t0)

        np_step()
        call_times.clear()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            np_step()
        wall = time.perf_counter() - t0
        h2d = sum(shard.count * D * (8 if p == "double" else 4) for p in precs for _ in fns)
        d2h = sum(shard.count * (8 if p == "double" else 4) for p in precs for _ in fns)
        e2e_numpy = {"value": args.steps * len(fns) * len(precs) * args.n / wall, "unit": UNIT,
                     "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                     "ms_per_step": 1e3 * wall / args.steps,
                     "path": ("Engine.evaluate(fn, numpy float64 X, precision) -> rb_h_func_evaluate[f]; "
                              "float32 calls cast X on the host first, as the reference does (engine.py:201)"),
                     "timing": "host wall clock around the blocking calls"}
        # the same step through the many-call host API: one population, every
        # (function, precision) in ONE call (rb_h_func_evaluate_many): the
        # rows cross PCIe once per step instead of once per call
        if args.config == 5:
            engine.evaluate_many(calls, xh)
            t0 = time.perf_counter()
            for _ in range(args.steps):
                engine.evaluate_many(calls, xh)
            wall_m = time.perf_counter() - t0
            e2e_numpy["many_call"] = {
                "value": args.steps * len(calls) * args.n / wall_m, "unit": UNIT,
                "h2d_bytes_per_step": shard.count * D * 8,
                "d2h_bytes_per_step": sum(shard.count * (8 if p == "double" else 4) for _, p in calls),
                "ms_per_step": 1e3 * wall_m / args.steps,
                "path": ("Engine.evaluate_many([(fn, precision) ...], numpy float64 X) -> "
                         "rb_h_func_evaluate_many: X uploaded once per ~32 MB row chunk for all "
                         "calls, float32 cast on the device"),
                "timing": "host wall clock around the blocking call"}
        if args.config == 1:
            dev_us = sorted(1e3 * a.elapsed_time(b) / r for evs in per.values() for a, b, r in evs)
            latency = {"device_us_per_call_median": dev_us[len(dev_us) // 2],
                       "host_blocking_us_per_call_median": 1e6 * statistics.median(call_times),
                       "calls": len(call_times),
                       "note": "device: one evaluation of N=1000 rows back to back (CUDA events "
                               "around 8 calls queued together); host: the whole blocking NumPy "
                               "call (validation, H2D, kernel, D2H)"}
            latency["graph"] = graph_latency(engine, fns[0], precs[0], xrot, stream)
        del xh

    # e2e through the public API from pinned host memory (config 5)
    e2e = None
    if not args.no_e2e and args.config == 5:
        host_x = torch.empty((shard.count, D), dtype=torch.float64, pin_memory=True)
        host_x.copy_(x64)
        host_f = torch.empty(args.n, dtype=torch.float64, pin_memory=True)
        dev_x = x64   # overwritten in place by each step's H2D copy (same values)
        h2d = shard.count * D * 8
        d2h = 0

        def e2e_step_plain():
            # N > 1 GPUs: this rank's rows in, every function's full N-vector
            # (after the all-gather) out, evaluations queued without a host
            # synchronisation per call (dist.ShardedEngine.submit)
            nonlocal d2h
            d2h = 0
            dev_x.copy_(host_x, non_blocking=True)
            x32e = dev_x.float()
            pend = []
            for p in precs:
                xe = dev_x if p == "double" else x32e
                for fn in fns:
                    k = len(pend)
                    if k >= 2:
                        stream.wait_event(pend[k - 2].done)
                    pd = sharded.submit(fn, xe, p, local_out=local_bufs[p][k % 2], out=full_bufs[p][k % 2])
                    stream.wait_event(pd.done)
                    full = pd.values
                    dst = host_f[: full.numel()] if p == "double" else host_f.view(torch.float32)[: full.numel()]
                    dst.copy_(full, non_blocking=True)
                    d2h += full.numel() * full.element_size()
                    pend.append(pd)
            torch.cuda.synchronize()
            check(pend)

        # one GPU: a chunked pipeline -- the H2D copy of row chunk c+1 and the
        # D2H of chunk c-1's fitness values run on a copy stream while chunk c
        # is evaluated (every function, both precisions; values land in a
        # resident results buffer through Engine.evaluate(out=...))
        n_chunks = int(os.environ.get("RB_E2E_CHUNKS", "8"))
        n_chunks = n_chunks if world == 1 and shard.count >= n_chunks * 4096 else 1
        # RB_E2E_TAPER=1: small first / last chunks (shorter pipeline fill
        # -- the first H2D -- and drain -- the last D2H)
        wts = [1] * n_chunks
        if os.environ.get("RB_E2E_TAPER", "1") == "1" and n_chunks >= 6:
            wts = [1, 4] + [8] * (n_chunks - 4) + [4, 1]
        cum = np.cumsum([0] + wts)
        bounds = [int(shard.count * int(c) // int(cum[-1])) for c in cum]
        nc_max = max(bounds[c + 1] - bounds[c] for c in range(n_chunks))
        copy_stream = torch.cuda.Stream(device=dev)     # H2D
        out_stream = torch.cuda.Stream(device=dev)      # D2H (PCIe is full duplex)
        res, host_res = {}, {}
        if world == 1:                    # resident results of two chunks in flight
            # slot layout [2][len(fns) * nc_max]: chunk c's values for function i
            # at [i * nc, (i + 1) * nc), so the D2H of a chunk is one contiguous
            # copy whatever its length
            res = {p: torch.empty((2, len(fns) * nc_max), device=dev,
                                  dtype=torch.float64 if p == "double" else torch.float32) for p in precs}
            host_res = {p: torch.empty((2, len(fns) * nc_max), dtype=res[p].dtype, pin_memory=True)
                        for p in precs}

        def e2e_step_pipelined():
            nonlocal d2h
            d2h = 0
            ev_in = [torch.cuda.Event() for _ in range(n_chunks)]
            ev_done = [torch.cuda.Event() for _ in range(n_chunks)]
            ev_out = [torch.cuda.Event() for _ in range(n_chunks)]
            with torch.cuda.stream(copy_stream):
                for c in range(n_chunks):
                    lo_, hi_ = bounds[c], bounds[c + 1]
                    dev_x[lo_:hi_].copy_(host_x[lo_:hi_], non_blocking=True)
                    ev_in[c].record(copy_stream)
            pend = []
            for c in range(n_chunks):
                lo_, hi_ = bounds[c], bounds[c + 1]
                nc = hi_ - lo_
                stream.wait_event(ev_in[c])
                if c >= 2:
                    stream.wait_event(ev_out[c - 2])        # results slot c % 2 copied out
                xc = dev_x[lo_:hi_]
                xcs = {"double": xc, "single": xc.float()}
                for p in precs:
                    for i, fn in enumerate(fns):
                        pend.append(engine.evaluate_async(fn, xcs[p], p,
                                                          out=res[p][c % 2, i * nc:(i + 1) * nc]))
                ev_done[c].record(stream)
                with torch.cuda.stream(out_stream):
                    out_stream.wait_event(ev_done[c])
                    for p in precs:
                        host_res[p][c % 2, :len(fns) * nc].copy_(res[p][c % 2, :len(fns) * nc],
                                                                  non_blocking=True)
                        d2h += len(fns) * nc * res[p].element_size()
                    ev_out[c].record(out_stream)
            stream.wait_stream(copy_stream)
            stream.wait_stream(out_stream)
            torch.cuda.synchronize()
            check(pend)

        e2e_step = e2e_step_pipelined if world == 1 else e2e_step_plain

        e2e_step()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        ems = a.elapsed_time(b)
        if world > 1:
            tt = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": evals / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / args.steps,
               "pipeline": (f"{n_chunks} row chunks (small first and last ones): H2D of X and D2H of every fitness vector on two "
                            "copy streams, overlapped with evaluation" if world == 1 else
                            "H2D, evaluations queued with their NCCL all-gathers overlapped, D2H per function")}
        del host_x, host_f, host_res, res

    e2e_pinned_tensor = None
    if e2e_many is not None:
        e2e_pinned_tensor, e2e = e2e, e2e_many
    if args.config != 5:
        e2e = e2e_numpy

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # all cores over min(N, --cpu-rows) rows, and one pinned core
        procs = os.cpu_count() or 1
        total = min(args.n, args.cpu_rows)
        per_proc = max(1, -(-total // procs))
        sample = x64[: per_proc * procs].cpu().numpy()                  # rows 0.. of X
        cpu = cpu_reference(D, fns, precs, per_proc, x_rows=sample, pin=True)
        one = cpu_reference(D, fns, precs, min(args.cpu_rows_1core, args.n), x_rows=sample,
                            procs=1, pin=True)
        cpu["single_core"] = {"value": one["value"], "unit": UNIT, "cores": 1,
                              "sample": one["sample"], "pinned": "core 0"}

    if args.breakdown and rank == 0:
        Path(args.breakdown).write_text(json.dumps({"rows": rows, "n_local": shard.count,
                                                    "dim": D}, indent=1))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64+f32" if len(precs) == 2 else ("f64" if precs[0] == "double" else "f32"),
            "data": ("synthetic X = numpy Philox(SeedSequence((0, D, N, 1001))).uniform(-100, 100), "
                     "drawn on the device bit-identically (population.py)"),
            "config": {"workload": (f"config {args.config}: {CONFIGS[args.config]['name']}"
                                    if args.config != 5 else
                                    f"suite-sweep D={D} N={args.n} ({len(fns)} fns x {len(precs)} precisions)"),
                       "baseline_config": args.config,
                       "dim": D, "n": args.n, "fns": len(fns), "precisions": precs,
                       "parallelism": f"rows/{world}", "l2": l2_note,
                       "seed": 0},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "e2e_pinned_tensor": e2e_pinned_tensor,
            "e2e_numpy": e2e_numpy if args.config == 5 else None, "latency": latency,
            "clocks": clk,
            "per_precision_evals_per_s": {
                p: len(fns) * args.n / sum(r["seconds"] for r in rows if r["precision"] == p)
                for p in precs},
        }
        print(json.dumps(line), flush=True)
    engine.dispose()
    if world > 1:
        dist.destroy_process_group()


def graph_latency(engine, fn, prec, xrot, stream, reps=64, rounds=9):
    """Config 1 through Engine.capture: the same N=1000 evaluation as CUDA
    graphs, one per rotating copy of X (so a replay reads X from HBM, not
    L2, as the timed steps do), replayed back to back -- one cudaGraphLaunch
    per evaluation, no per-call validation.  Device time per replay (CUDA
    events around ``reps`` replays on the launching stream) and host time
    for launch + wait + status of one replay."""
    import torch
    caps = [engine.capture(fn, xr[prec], prec) for xr in xrot]
    for c in caps:
        c.launch()
    for c in caps:
        c.result()
    dev, host = [], []
    k = 0
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            caps[k % len(caps)].launch()
            k += 1
        e1.record(stream)
        torch.cuda.synchronize()
        for c in caps:
            c.result()
        dev.append(1e3 * e0.elapsed_time(e1) / reps)
    for _ in range(reps):
        c = caps[k % len(caps)]
        k += 1
        t0 = time.perf_counter()
        c.launch().result()
        host.append(1e6 * (time.perf_counter() - t0))
    for c in caps:
        c.close()
    return {"device_us_per_call_median": statistics.median(dev),
            "evals_per_s": 1e6 * int(xrot[0][prec].shape[0]) / statistics.median(dev),
            "host_us_per_call_median": statistics.median(host),
            "graphs": len(caps),
            "note": "Engine.capture (rb_graph_capture): one graph per rotating X copy, one "
                    "cudaGraphLaunch per evaluation, queued back to back (bounded by the host cost "
                    "of cudaGraphLaunch when it exceeds the 6 us kernel); host = launch + wait + "
                    "status of one replay"}


def main():
    args = parse()
    maybe_spawn(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
