#!/usr/bin/env python
"""Benchmark of the B200 multigrid solve path (driver contract: one JSON line).

Metric (BASELINE.json): multigrid DOF*V-cycles/s to a relative residual of
1e-10, plus smoother/residual HBM GB/s.  A *step* is one full solve
(MultigridSolver::solve, u0 = 0 .. converged norm) of the workload:

  c3 (default)  256 Shafranov 513x512 sections, alpha scaled per section,
                sharded over the ranks (strong scaling, no collectives) --
                the largest single-GPU config and the scaling config
  c0            CirclePolar 257x256, Give, V(1,1)
  c1            Shafranov 1025x1024, Take, V(1,1)           (BASELINE configs[1])
  c2v / c2w     Czarny 4097x4096, Take, V(1,1) / W(1,1)
  c4            Czarny 8193x8192 kernel roofline microbench (Take residual,
                circle sweep B+W, radial sweep B+W; 100 reps each)

value: device time (CUDA events on the solver's stream, L2 flushed between
steps by a 512 MiB write) with the RHS already in HBM; e2e: the same solve
through the public C ABI from pinned host buffers (H2D of f and D2H of u inside
the timed region).  Multi-GPU: one process per GPU (torchrun), barrier +
synchronize around the timed region, max over ranks.
`--impl reference` times the reference's own CPU implementation
(oracle/_ref, all host threads) on the same workload.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20240611
METRIC = "multigrid DOF*V-cycles/sec to rel. residual 1e-10"
UNIT = "DOF*cycles/s"

WORKLOADS = {
    "c0": (0, "CirclePolar 257x256 Give V(1,1) rel 1e-10"),
    "c1": (1, "Shafranov 1025x1024 Take V(1,1) rel 1e-10"),
    "c2v": (2, "Czarny 4097x4096 Take V(1,1) rel 1e-10"),
    "c2w": (2, "Czarny 4097x4096 Take W(1,1) rel 1e-10"),
    "c3": (3, "256 x Shafranov 513x512 Take V(1,1) rel 1e-10, alpha*U(0.5,2)"),
    "c4": (4, "Czarny 8193x8192 Take kernel microbench"),
    "give": (2, "Czarny 4097x4096 Give kernel microbench"),
}

# algorithmic bytes per node of one launch
# (smooth: one zebra smoothing step = circle B+W over the circle nodes + radial
# B+W over the radial nodes = 56 B per node of the level)
BYTES_PER_NODE = {"residual": 56.0, "circle": 56.0, "radial": 56.0, "smooth": 56.0,
                  "restrict": 10.0, "prolongate": 18.0}


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sms, mx, reasons, loaded = [], None, set(), []
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm, smmax, util = float(parts[0]), float(parts[1]), float(parts[6])
            except ValueError:
                continue
            sms.append(sm)
            mx = smmax
            if util > 0:
                loaded.append(sm)
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        pool = loaded or sms
        return {"sm_mhz": statistics.median(pool) if pool else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms), "samples_loaded": len(loaded)}


# ---------------------------------------------------------------- reference
def ref_case(k: int, cycle: str = "V", **over):
    from oracle.oracle import config_case
    c = config_case(k, cycle=cycle, **over)
    return c


def _section_worker(args):
    """One sections-parallel worker (its own process, 1 OpenMP thread):
    builds the solvers of its sections (setup, untimed), warms up once, waits
    for every worker, then solves its sections back to back."""
    idx, barrier = args
    from oracle.oracle import RefSolver, section_scales as ref_scales
    scales = ref_scales(256)
    work = []
    for i in idx:
        R = RefSolver(ref_case(3, alpha_scale=float(scales[i]), threads=1))
        _, f = R.seeded_rhs(SEED + i)
        work.append((R, f))
    work[0][0].solve(work[0][1])  # in-process warm-up (first solve is slow)
    barrier.wait()
    t0 = time.perf_counter()
    units = 0.0
    for R, f in work:
        units += R.n(0) * R.solve(f)["iterations"]
    return t0, time.perf_counter(), units


def c3_sections_parallel(idx, procs):
    """`procs` sections concurrently at 1 thread each.
    Returns (DOF*cycles/s, wall seconds of the concurrent solve phase)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    barrier = mgr.Barrier(procs)
    chunks = [idx[p::procs] for p in range(procs)]
    with ctx.Pool(procs) as pool:
        res = pool.map(_section_worker, [(c, barrier) for c in chunks])
    mgr.shutdown()
    wall = max(r[1] for r in res) - min(r[0] for r in res)
    return sum(r[2] for r in res) / wall, wall


def c3_sequential(idx, threads):
    """the sections one after another, all threads each."""
    from oracle.oracle import RefSolver, section_scales as ref_scales
    scales = ref_scales(256)
    units = secs = 0.0
    for j, i in enumerate(idx):
        R = RefSolver(ref_case(3, alpha_scale=float(scales[i]), threads=threads))
        _, f = R.seeded_rhs(SEED + i)
        if j == 0:
            R.solve(f)  # warm-up
        out = R.solve(f)
        units += R.n(0) * out["iterations"]
        secs += out["seconds"]
    return units / secs, secs


def cpu_reference_solves(workload: str, n_solves: int, warm: int = 1, sections=None,
                         c3_mode=None):
    """Times the reference polarmg solve (oracle/_ref) on the workload; returns
    (DOF*cycles/s, seconds, solves, sample description, threads, c3 mode).

    Config 3 is timed both ways -- `threads` sections at once
    with 1 OpenMP thread each, and the same sections one after another with
    `threads` threads each -- and the better is reported (c3_mode pins one)."""
    from oracle.oracle import RefSolver
    k, _ = WORKLOADS[workload]
    cycle = "W" if workload == "c2w" else "V"
    threads = os.cpu_count() or 1
    if k == 3:
        idx = sections if sections is not None else list(range(min(n_solves, 256)))
        modes = {}
        if c3_mode in (None, "sections-parallel"):
            modes["sections-parallel"] = c3_sections_parallel(idx, min(threads, len(idx)))
        if c3_mode in (None, "sequential"):
            modes["sequential"] = c3_sequential(idx, threads)
        best = max(modes, key=lambda m: modes[m][0])
        v, secs = modes[best]
        both = ", ".join(f"{m} {modes[m][0]:.3e}" for m in modes)
        sample = (f"sections {idx[0]}..{idx[-1]} ({len(idx)} of 256), {best} "
                  f"({both} DOF*cycles/s)")
        return v, secs, len(idx), sample, threads, best
    R = RefSolver(ref_case(k, cycle=cycle, threads=threads))
    _, f = R.seeded_rhs(SEED)
    for _ in range(warm):
        R.solve(f)
    units = secs = 0.0
    count = 0
    for _ in range(n_solves):
        out = R.solve(f)
        units += R.n(0) * out["iterations"]
        secs += out["seconds"]
        count += 1
    sample = f"{count} full solves of {WORKLOADS[workload][1]} after {warm} warm-up"
    return units / secs, secs, count, sample, threads, None


def config_dict(workload, world):
    """The `config` object both arms print (same keys and values)."""
    k, desc = WORKLOADS[workload]
    geo = {0: "257x256", 1: "1025x1024", 2: "4097x4096", 3: "513x512", 4: "8193x8192"}[k]
    cfg = {"workload": f"{workload}: {desc}", "grid": geo,
           "sections": 256 if k == 3 else 1,
           "l2": "flushed between steps (512 MiB write, untimed)",
           "parallelism": (f"{world} ranks, 256 sections sharded contiguously, no collectives"
                           if k == 3 else f"{world} independent replicas, no collectives")}
    return cfg


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    wl = args.workload
    if wl in ("c4", "give"):
        print(json.dumps({"impl": "reference",
                          "unavailable": f"{wl} is a kernel microbench; use c3"}))
        return 0
    threads = os.cpu_count() or 1
    per_step = []
    units_total = 0.0
    samples = []
    c3_mode = None
    for step in range(args.warmup + args.steps):
        if wl == "c3":
            # a bounded sample per step: `threads` consecutive sections
            cnt = min(threads, 256)
            first = (step * cnt) % 256
            idx = [(first + j) % 256 for j in range(cnt)]
            v, secs, _, sample, threads, mode = cpu_reference_solves(
                wl, cnt, sections=idx, c3_mode=c3_mode)
            if step == 0:
                c3_mode = mode  # the better mode, measured on the first warm-up step
        else:
            v, secs, _, sample, threads, _ = cpu_reference_solves(wl, 1, warm=0 if step else 1)
        if step >= args.warmup:
            per_step.append(secs)
            units_total += v * secs
            samples.append(sample)
    total = sum(per_step)
    value = units_total / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong" if wl == "c3" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded U(-1,1) u*, f = A u*)",
        "config": config_dict(wl, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{args.steps} steps; step 1: {samples[0]}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------- GPU
def build_solver(workload, rank, world, stream, reference_order=True, device=0):
    import paper_2507_03812_b200 as pmg
    k, _ = WORKLOADS[workload]
    cyc = "W" if workload == "c2w" else "V"
    geom, prob, grid, st, meta = pmg.baseline_config(k, cycle=cyc,
                                                     reference_order=reference_order)
    sections = None
    if k == 3:
        from paper_2507_03812_b200.shard import section_shard
        scales = pmg.section_scales(256)
        sections = section_shard(256, rank, world)
        solver = pmg.MultigridSolver(geom, prob, grid, st, n_sections=len(sections),
                                     alpha_scales=scales[sections], device=device,
                                     stream=stream)
    else:
        solver = pmg.MultigridSolver(geom, prob, grid, st, device=device, stream=stream)
    return solver, sections


def seeded(solver, workload, rank, sections):
    if sections is not None:
        # per-section seeds SEED + global index: seed the batch at its first index
        solver.seeded_rhs(SEED + sections[0])
    else:
        solver.seeded_rhs(SEED + rank)


def run_gpu(args):
    import torch
    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    peak, peak_kind = peaks()

    if args.workload == "c4":
        return run_c4(args, rank, world, local, stream, peak, peak_kind, dist)
    if args.workload == "give":
        return run_give(args, rank, world, local, stream, peak, peak_kind, dist)

    # --rank-slice N (one process, one GPU): run only the slice rank 0 of an
    # N-GPU job would own -- the per-rank workload of the sharded batch, which
    # has no inter-GPU dependence, so N such ranks finish in max-over-ranks of
    # this time; a projection aid where only one GPU is available
    shard_world = args.rank_slice if (args.rank_slice > 1 and world == 1) else world
    solver, sections = build_solver(args.workload, rank, shard_world, stream.cuda_stream,
                                    not args.fast, device=local)
    seeded(solver, args.workload, rank, sections)
    n = solver.n(0)
    B = solver.n_sections
    flush = torch.empty(64 << 20, dtype=torch.float64, device=dev)  # 512 MiB > 126 MB L2

    def one_solve():
        rep = solver.solve()
        its = [r.iterations for r in solver.reports]
        return rep, its

    for _ in range(args.warmup):
        flush.add_(1.0)
        one_solve()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = solver.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    units = 0.0
    iters = None
    for i in range(args.steps):
        flush.add_(1.0)
        starts[i].record(stream)
        rep, its = one_solve()
        ends[i].record(stream)
        units += float(n) * sum(its)
        iters = its
    torch.cuda.synchronize()
    launches = solver.launch_count() - l0
    clk = clocks.stop()
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    if dist:
        t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
        u = torch.tensor([units], dtype=torch.float64, device=dev)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
        units = float(u.item())
    value = units / (dev_ms * 1e-3)

    # ---- e2e: public API from pinned host buffers (H2D f, solve, D2H u)
    import ctypes
    f_host = torch.empty(B * n, dtype=torch.float64, pin_memory=True)
    u_host = torch.empty(B * n, dtype=torch.float64, pin_memory=True)
    f_host.numpy()[:] = solver.get_rhs()
    fptr = ctypes.cast(f_host.data_ptr(), ctypes.POINTER(ctypes.c_double))
    uptr = ctypes.cast(u_host.data_ptr(), ctypes.POINTER(ctypes.c_double))
    e2e_steps = max(3, min(args.steps, 10))
    e2e_units = 0.0
    e2e_total = 0.0
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    for _ in range(e2e_steps):
        flush.add_(1.0)
        torch.cuda.synchronize()
        a = time.perf_counter()
        rc1 = solver._lib.pmg_set_rhs(solver._h, fptr, 0)
        rep, its = one_solve()
        rc2 = solver._lib.pmg_get_solution(solver._h, uptr, 0)
        e2e_total += time.perf_counter() - a
        assert rc1 == 0 and rc2 == 0
        e2e_units += float(n) * sum(its)
    if dist:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
        u = torch.tensor([e2e_units], dtype=torch.float64, device=dev)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
        e2e_units = float(u.item())
    e2e_value = e2e_units / e2e_total

    # ---- per-kernel-class breakdown of one solve (CUDA events per launch)
    solver.profile(True)
    flush.add_(1.0)
    one_solve()
    breakdown = {}
    for kind in ("residual", "smooth", "circle", "radial", "restrict", "prolongate", "coarse",
                 "norm", "other"):
        ms, cnt = solver.profile_read(kind)
        if cnt:
            breakdown[kind] = {"ms": round(ms, 4), "launches": cnt}
    solver.profile(False)
    # "smooth" = fused smoothing steps (all four zebra sweeps of a level in one
    # launch, the latency-bound levels); circle / radial = per-colour sweeps
    dominant = max(("residual", "smooth", "circle", "radial"),
                   key=lambda k: breakdown.get(k, {"ms": 0})["ms"])

    # ---- roofline of the dominant kernel on the finest level
    roof = kernel_roofline(solver, dominant, peak, peak_kind, reps=20, workload=args.workload)
    kernels = {k: kernel_roofline(solver, k, peak, peak_kind, reps=20, workload=args.workload)
               for k in ("residual", "smooth", "circle", "radial")}

    # which CUDA device each rank's solver ran on (LOCAL_RANK by construction)
    devices = [local]
    if dist:
        got = [None] * world
        dist.all_gather_object(got, local)
        devices = got
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            if args.workload == "c3":
                thr = os.cpu_count() or 1
                v, secs, cnt, sample, thr, _ = cpu_reference_solves(
                    "c3", thr, sections=list(range(min(8 * thr, 256))))  # ~10-20 s of CPU work
            else:
                ns = 2 if args.workload in ("c1", "c0") else 1
                v, secs, cnt, sample, thr, _ = cpu_reference_solves(args.workload, ns)
            cpu = {"value": v, "unit": UNIT, "cores": thr, "kind": "reference",
                   "sample": sample + f" ({secs:.1f} s of CPU solve time)"}
        except Exception as e:  # the checker must not mask a GPU result
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    nr, nt, split = solver.level_shape(0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.workload == "c3" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded U(-1,1) u*, f = A u*; random-free grid)",
        "config": config_dict(args.workload, world),
        "run_info": {"grid": f"{nr}x{nt}", "split": split, "levels": solver.num_levels(),
                     "sections_per_rank": B, "devices": devices,
                     "rank_slice_of": args.rank_slice if args.rank_slice > 1 else None,
                     "iterations_first_sections": iters[:4] if iters else None,
                     "line_solves": "reference order (bitwise)" if not args.fast
                     else "chunked parallel scans"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * B * n,
                "d2h_bytes_per_step": 8 * B * n, "steps": e2e_steps,
                "timer": "host wall clock around set_rhs + solve + get_solution"},
        "gpu_launches": launches,
        "clocks": clk,
        "breakdown_one_solve": breakdown,
        "kernels_finest_level": kernels,
    }
    if args.workload == "c3" and world == 1 and not args.no_extras and args.rank_slice <= 1:
        # the single-grid config 2 (4097x4096, V and W cycles) beside the headline
        solver.close()
        line["extra"] = {w: single_grid_line(w, stream, local, torch, flush, not args.fast)
                         for w in ("c2v", "c2w")}
    print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def single_grid_line(workload, stream, local, torch, flush, reference_order, solves=2):
    """Device-timed solves (1 warm-up + `solves`, L2 flushed between) of a
    single-grid config: DOF*cycles/s, ms per solve, iterations."""
    solver, _ = build_solver(workload, 0, 1, stream.cuda_stream, reference_order, device=local)
    seeded(solver, workload, 0, None)
    n = solver.n(0)
    ms, its = [], 0
    for i in range(1 + solves):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rep = solver.solve()
        b.record(stream)
        torch.cuda.synchronize()
        if i:
            ms.append(a.elapsed_time(b))
        its = rep.iterations
    solver.close()
    t = sum(ms) / len(ms)
    return {"workload": WORKLOADS[workload][1], "value": n * its / (t * 1e-3), "unit": UNIT,
            "ms_per_solve": round(t, 3), "iterations": its, "solves": solves}


def ncu_traffic(workload, kind):
    """DRAM bytes per launch (B+W pair for sweeps) of the finest-level kernel
    from the committed ncu capture (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(workload, {}).get(kind)
    except Exception:
        return None


def kernel_roofline(solver, kind, peak, peak_kind, reps=20, workload=None):
    """achieved = algorithmic bytes per launch / CUDA-event time per launch on
    the finest level (L2 flushed before every repetition)."""
    nr, nt, split = solver.level_shape(0)
    B = solver.n_sections
    if kind in ("residual", "smooth"):
        nodes = nr * nt
    elif kind == "circle":
        nodes = split * nt
    else:
        nodes = (nr - split) * nt
    if nodes == 0:
        return None
    ms = solver.time_kernel(kind, 0, reps, True)
    algo = BYTES_PER_NODE[kind] * nodes * B
    gbs = algo / (ms * 1e-3) / 1e9
    label = {"residual": "", "smooth": ", circle B+W + radial B+W"}.get(kind, ", B+W")
    return {"kernel": f"{kind} (finest level{label})",
            "bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
            "frac": round(gbs / peak, 4), "traffic": ncu_traffic(workload, kind),
            "ms_per_launch": round(ms, 5),
            "algorithmic_bytes": algo, "bytes_per_node": BYTES_PER_NODE[kind],
            "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"}


# Give mode (stencil.cpp:176-287 recast as a gather): coefficients are
# re-evaluated on the fly, so a launch moves only u, f and the result (24 B per
# node); the sweeps also read their two factor bands (40 B).  The
# FP64 operations per node are counted by ncu (smsp__sass_thread_inst_executed_
# op_d{fma,mul,add}_pred_on of the captures under profiles/; 2 flops per DFMA)
# and reported against the B200's FP64 vector peak next to the HBM fraction.
GIVE_BYTES = {"residual": 24.0, "circle": 40.0, "radial": 40.0}
FP64_PEAK_TFLOPS = 37.0  # datasheet FP64 (non-tensor) peak; not in MEASURED_PEAKS.json


def run_give(args, rank, world, local, stream, peak, peak_kind, dist):
    """Give-operator roofline at 4097x4096: residual,
    circle sweep B+W and radial sweep B+W against HBM and FP64 peak."""
    import paper_2507_03812_b200 as pmg
    geom, prob, grid, st, meta = pmg.baseline_config(2, stencil_mode="Give",
                                                     reference_order=not args.fast)
    solver = pmg.MultigridSolver(geom, prob, grid, st, device=local, stream=stream.cuda_stream)
    n = solver.n(0)
    nr, nt, split = solver.level_shape(0)
    rng = np.random.default_rng(SEED)
    solver.residual(rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), 0)
    try:
        with open(os.path.join(ROOT, "profiles", "give_flops.json")) as fh:
            flops = json.load(fh)
    except Exception:
        flops = {}
    out = {}
    for k in ("residual", "circle", "radial"):
        nodes = {"residual": nr * nt, "circle": split * nt, "radial": (nr - split) * nt}[k]
        ms = solver.time_kernel(k, 0, args.reps, True)
        gbs = GIVE_BYTES[k] * nodes / (ms * 1e-3) / 1e9
        fl = flops.get(k)  # FP64 flops per node (ncu)
        out[k] = {"kernel": f"Give {k} (finest level{'' if k == 'residual' else ', B+W'})",
                  "ms_per_launch": round(ms, 5), "bytes_per_node": GIVE_BYTES[k],
                  "hbm": {"achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                          "frac": round(gbs / peak, 4)},
                  "fp64": None if fl is None else {
                      "flops_per_node": fl, "achieved": round(fl * nodes / (ms * 1e-3) / 1e12, 2),
                      "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                      "frac": round(fl * nodes / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4)}}
    if rank == 0:
        print(json.dumps({"metric": "Give residual/smoother GB/s and FP64 TFLOP/s (4097x4096)",
                          "value": out["residual"]["hbm"]["achieved"], "unit": "GB/s",
                          "n_gpus": world, "steps": args.reps, "warmup": 0,
                          "higher_is_better": True, "dtype": "f64",
                          "config": {"workload": "give: " + WORKLOADS["give"][1],
                                     "grid": "4097x4096",
                                     "l2": "flushed before every repetition"},
                          "kernels": out}))
    return 0


def run_c4(args, rank, world, local, stream, peak, peak_kind, dist):
    """Config 4 roofline microbench: 100 reps of the Take residual, circle
    sweep B+W and radial sweep B+W on seeded U(-1,1) iterates."""
    import paper_2507_03812_b200 as pmg
    geom, prob, grid, st, meta = pmg.baseline_config(4, reference_order=not args.fast)
    solver = pmg.MultigridSolver(geom, prob, grid, st, device=local, stream=stream.cuda_stream)
    n = solver.n(0)
    rng = np.random.default_rng(SEED)
    # u, f ~ U(-1,1): load through the operator seams' buffers
    u = rng.uniform(-1, 1, n)
    f = rng.uniform(-1, 1, n)
    solver.residual(u, f, 0)  # uploads u, f into level-0 buffers
    reps = args.reps
    out = {}
    for k in ("residual", "circle", "radial"):
        out[k] = kernel_roofline(solver, k, peak, peak_kind, reps=reps, workload="c4")
    if rank == 0:
        line = {"metric": "smoother/residual HBM GB/s (config 4 microbench)",
                "value": out["radial"]["achieved"], "unit": "GB/s", "n_gpus": world,
                "steps": reps, "warmup": 0, "higher_is_better": True, "dtype": "f64",
                "config": {"workload": "c4: " + WORKLOADS["c4"][1], "grid": "8193x8192",
                           "l2": "flushed before every repetition",
                           "line_solves": "chunked scans (fast)" if args.fast
                           else "reference order (bitwise)"},
                "kernels": out}
        print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--workload", default="c3", choices=list(WORKLOADS))
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rank-slice", type=int, default=0,
                    help="c3 on one GPU: only the sections rank 0 of an N-GPU job owns")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the config-2 V/W lines added to the default c3 run")
    # default: line solves bitwise the reference's (the parity contract);
    # --fast: chunked parallel scans (roundoff-level drift from the reference)
    ap.add_argument("--fast", action="store_true")
    ap.add_argument("--reference-order", action="store_true", help="(default; kept for scripts)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "gpu":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu(args)


def spawn_ranks(n):
    """`--gpus N` outside torchrun: launch N ranks (one process per GPU) the
    way the driver does and return rank 0's exit status."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
