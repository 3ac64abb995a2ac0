#!/usr/bin/env python
"""Benchmark of the ADI hp-FEM solve (arXiv 2402.11299 hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5]

One step = hpfem_load (F_leg -> G, K8) + hpfem_solve (G -> U: 2J fused
half-steps + the final W_J C^{-1}) on one synthetic right-hand side of the
configuration (default: BASELINE.json configs[4], the largest, on which the
north_star's HBM bar is set).  Inputs are resident in HBM when the timed
region starts; every array (2.15 GB) exceeds L2 (126 MB), so no L2 flush is
needed.  Time is taken with CUDA events on the launch stream around exactly
K steps bracketed by barrier + synchronize, max over ranks.

N > 1 runs N independent replicas (one per GPU, "replicas only": the path
has no exchange step); value = N*K / max-rank time.

--impl reference times the CPU oracle (oracle/, the deliberately slow
baseline) on the host cores on a bounded sample of the same workload
(load + 1 of the J ADI iterations + final, scaled to a full solve).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADI Poisson solves/s and DOF/s (fp64) at 1 B200; achieved HBM GB/s vs peak"


# --------------------------------------------------------------- multi-rank
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reduce_max(x: float, backend_device=None) -> float:
    """Max over ranks (identity when torch.distributed is not initialised)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=backend_device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(world: int, steps: int, t_max_s: float) -> float:
    """Whole-job throughput: all solves of all ranks / max-rank time."""
    return world * steps / t_max_s


def barrier():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", self.gpu_id], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def gpu_id_for(dev: int) -> str:
    import torch

    try:
        u = str(torch.cuda.get_device_properties(dev).uuid)
        return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        return vis.split(",")[dev] if vis else str(dev)


# --------------------------------------------------------------- helpers
def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(cfg_idx: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the
    dominant kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            d = json.load(fh)
        return d[f"config{cfg_idx}"]["dram_bytes_per_launch"], d[f"config{cfg_idx}"].get("source")
    except Exception:
        return None, None


def _oracle_sample(cfg, Fleg, J):
    """Time the oracle as it stands on the host cores: a full load + solve
    when that takes well under ~20 s, else load + ADI solves with 1 and 3 of
    the J iterations, extrapolated to all J (the plan and the final
    W C^{-1} are in both samples and cancel in the per-iteration slope)."""
    import oracle

    xs, ys = cfg.breakpoints()
    oracle.build()
    t0 = time.perf_counter()
    G = oracle.load(xs, cfg.px, ys, cfg.py, cfg.bc, Fleg)
    t_load = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.adi_solve(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol, G, iters=1)
    t1 = time.perf_counter() - t0
    if t1 * J < 15.0:
        t0 = time.perf_counter()
        oracle.adi_solve(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol, G)
        t_full = t_load + time.perf_counter() - t0
        return t_full, f"config {cfg.idx}: full oracle load + solve (J={J}) timed: {t_full:.2f}s"
    t0 = time.perf_counter()
    oracle.adi_solve(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol, G, iters=3)
    t3 = time.perf_counter() - t0
    t_iter = max((t3 - t1) / 2, 1e-9)
    t_full = t_load + t1 + (J - 1) * t_iter
    return t_full, (f"config {cfg.idx}: oracle load ({t_load:.2f}s) + ADI solves with 1 and 3 of J={J} iterations "
                    f"({t1:.2f}s, {t3:.2f}s); full solve = load + t1 + (J-1)(t3-t1)/2 = {t_full:.1f}s")


def cpu_baseline(cfg, Fleg, J):
    """The oracle as it stands on the host cores: ONE measured full load +
    solve of the workload on all cores (config 5: ~3.5 min on 16 cores), and
    a single-threaded figure scaled from a measured 1-iteration sample (the
    per-thread cost ratio of the same 1-iteration solve on 1 and on all
    cores times the measured full run)."""
    import oracle

    xs, ys = cfg.breakpoints()
    oracle.build()
    oracle.set_threads(0)
    cores = oracle.threads()
    t0 = time.perf_counter()
    G = oracle.load(xs, cfg.px, ys, cfg.py, cfg.bc, Fleg)
    t_load = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, Jo = oracle.adi_solve(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol, G)
    t_full = t_load + time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.adi_solve(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol, G, iters=1)
    t1m = time.perf_counter() - t0
    oracle.set_threads(1)
    try:
        t0 = time.perf_counter()
        oracle.adi_solve(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol, G, iters=1)
        t1s = time.perf_counter() - t0
    finally:
        oracle.set_threads(0)
    t_single = t_full * t1s / t1m
    return {"value": 1.0 / t_full, "unit": "solves/s", "cores": cores, "kind": "oracle",
            "sample": (f"config {cfg.idx}: one full oracle load + solve (J={Jo}) measured on {cores} threads: "
                       f"{t_full:.1f}s (load {t_load:.1f}s)"),
            "measured_solve_s": t_full,
            "single_thread": {"value": 1.0 / t_single, "unit": "solves/s", "cores": 1,
                              "sample": (f"1-iteration solve measured on 1 thread {t1s:.1f}s vs {cores} threads "
                                         f"{t1m:.1f}s; full solve on 1 thread ~ {t_full:.1f}s x {t1s / t1m:.2f} "
                                         f"= {t_single:.0f}s")}}


# --------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    import workloads as W

    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle

    oracle.build()
    xs, ys = cfg.breakpoints()
    Fleg = W.f_leg(cfg, seed=0)
    J = oracle.plan(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol)["J"]

    for _ in range(args.warmup):
        _oracle_sample(cfg, Fleg, J)
    est, samples = [], []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t_full, sample = _oracle_sample(cfg, Fleg, J)
        est.append(t_full)
        samples.append(sample)
    wall = time.perf_counter() - t_start
    tmean = sum(est) / len(est)
    value = 1.0 / tmean
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmean * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{cfg.idx}:{cfg.name}", "N_x": cfg.Nx, "N_y": cfg.Ny, "J": J,
                   "dofs": cfg.dofs},
        "dof_per_s": value * cfg.dofs,
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": oracle.threads(), "kind": "oracle",
                         "sample": f"each step: {samples[-1]}; {len(est)} steps, sampled wall {wall:.1f}s"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2402_11299_b200 as hp
    import workloads as W

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    stream = torch.cuda.current_stream()
    xs, ys = cfg.breakpoints()
    Fleg = W.f_leg(cfg, seed=0)
    Fh = torch.from_numpy(Fleg).pin_memory()
    t0 = time.perf_counter()
    plan = hp.Plan(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol)
    plan_ms = (time.perf_counter() - t0) * 1e3
    Nx, Ny, J = plan.Nx, plan.Ny, plan.J
    Fd = Fh.to(f"cuda:{dev}")
    Gd = torch.empty((Nx, Ny), dtype=torch.float64, device=dev)
    Ud = torch.empty_like(Gd)
    Uh = torch.empty((Nx, Ny), dtype=torch.float64).pin_memory()

    def step():
        plan.load(Fd, Gd)
        plan.solve(Gd, Ud)

    launches_per_step = 0
    for _ in range(args.warmup):
        plan.load(Fd, Gd)
        launches_per_step = plan.launches()
        plan.solve(Gd, Ud)
        launches_per_step += plan.launches()
    torch.cuda.synchronize()

    # ---- device-resident timed region (events between the steps only)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(gpu_id_for(dev)) as clk:
        barrier()
        torch.cuda.synchronize()
        evs[0].record(stream)
        for k in range(args.steps):
            step()
            evs[k + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
    t_ms = evs[0].elapsed_time(evs[-1])
    step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    clocks = clk.summary()
    # ---- per-kernel-kind durations for the roofline: the same steps again with
    # CUDA events around every launch, on the launch stream, in the timed
    # configuration (the side-stream hat lines still run concurrently with
    # the bubble kernels; only the CUDA graph replay is off)
    plan.profile((12 * J + 32) * args.steps + 64)
    for _ in range(args.steps):
        step()
    prof = plan.profile_read()
    plan.profile(0)
    t_max_s = reduce_max(t_ms / 1e3, f"cuda:{dev}" if ws > 1 else None)
    value = job_value(ws, args.steps, t_max_s)
    ms_per_step = t_max_s * 1e3 / args.steps

    # ---- end-to-end through the public API with host buffers: every step
    # copies its F_leg from pinned host memory and its U back; the copies of
    # neighbouring steps run on two copy streams, overlapped with the current
    # step's compute (double-buffered device F_leg / U, pinned host U)
    e2e = None
    if not args.no_e2e:
        h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
        Fdb = [Fd, torch.empty_like(Fd)]
        Udb = [Ud, torch.empty_like(Ud)]
        Uhb = [Uh, torch.empty_like(Uh).pin_memory()]
        ev = lambda: torch.cuda.Event()

        def e2e_run(nsteps):
            loaded = [ev(), ev()]   # the load of the step that last read Fdb[b] is done
            copied = [ev(), ev()]   # the D2H that last read Udb[b] is done
            arrived = [ev(), ev()]  # the H2D into Fdb[b] is done
            solved = [ev(), ev()]
            for b in range(2):
                loaded[b].record(stream)
                copied[b].record(stream)
            with torch.cuda.stream(h2d):
                h2d.wait_event(loaded[0])
                Fdb[0].copy_(Fh, non_blocking=True)
                arrived[0].record(h2d)
            for k in range(nsteps):
                b = k & 1
                if k + 1 < nsteps:  # prefetch the next step's input
                    with torch.cuda.stream(h2d):
                        h2d.wait_event(loaded[b ^ 1])
                        Fdb[b ^ 1].copy_(Fh, non_blocking=True)
                        arrived[b ^ 1].record(h2d)
                stream.wait_event(arrived[b])
                plan.load(Fdb[b], Gd)
                loaded[b].record(stream)
                stream.wait_event(copied[b])
                plan.solve(Gd, Udb[b])
                solved[b].record(stream)
                with torch.cuda.stream(d2h):
                    d2h.wait_event(solved[b])
                    Uhb[b].copy_(Udb[b], non_blocking=True)
                    copied[b].record(d2h)
            stream.wait_stream(h2d)
            stream.wait_stream(d2h)

        e2e_run(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        e2e_run(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        te = reduce_max(e0.elapsed_time(e1) / 1e3, f"cuda:{dev}" if ws > 1 else None)
        e2e = {"value": job_value(ws, args.steps, te), "unit": "solves/s",
               "h2d_bytes_per_step": int(Fh.numel() * 8), "d2h_bytes_per_step": int(Uh.numel() * 8),
               "ms_per_step": te * 1e3 / args.steps,
               "copies": "per step: F_leg H2D from pinned host + U D2H to pinned host, on two copy streams "
                         "overlapping the neighbouring steps' compute (double-buffered)"}

    # ---- roofline of the dominant kernel (half-step bubble kernel K2-K4)
    peak, peak_kind = measured_peak()
    kb = {k: prof["halfstep_bubbles_x"][k] + prof["halfstep_bubbles_y"][k] for k in ("ms", "launches", "bytes")}
    pth = plan.path()
    kernel_label = {
        "tma": "k_xstep_tma / k_ystep_tma (K2: TMA-fed half-step kernels, fused apply + bubble-chain solve)"
               + (", transposed solve" if pth["transposed"] else ""),
        "ldg": "k_bubbles<0> / k_bubbles<1> (K2, LDG streaming variant)",
        "small": "k_adi_small (K11: whole solve in one CTA; no per-kernel times)",
    }.get(pth["path"], str(pth["path"]))
    achieved = kb["bytes"] / (kb["ms"] / 1e3) / 1e9 if kb["ms"] > 0 else None
    traffic, traffic_src = ncu_traffic(cfg.idx)
    total_kernel_ms = sum(v["ms"] for v in prof.values())
    alg_bytes_step = 8.0 * Nx * Ny * (6 * J + 1)
    roofline = {
        "bound": "hbm", "kernel": kernel_label,
        "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": (achieved / peak) if achieved else None, "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
        "traffic": traffic, "traffic_source": traffic_src,
        "launches": kb["launches"], "avg_launch_ms": kb["ms"] / max(kb["launches"], 1),
        "share_of_step": kb["ms"] / total_kernel_ms if total_kernel_ms else None,
        "solve_alg_GBps": alg_bytes_step / (ms_per_step / 1e3) / 1e9,
        "solve_alg_frac": alg_bytes_step / (ms_per_step / 1e3) / 1e9 / peak,
        "per_kind_ms": {k: round(v["ms"] / args.steps, 4) for k, v in prof.items()},
        "per_direction": {d: {"avg_launch_ms": v["ms"] / max(v["launches"], 1), "launches": v["launches"],
                              "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 else None,
                              "frac": v["bytes"] / (v["ms"] / 1e3) / 1e9 / peak if v["ms"] > 0 else None}
                          for d, v in (("x_solves", prof["halfstep_bubbles_x"]), ("y_solves", prof["halfstep_bubbles_y"]))},
        "per_kind_source": ("CUDA events around every launch on the launch stream, in the timed configuration "
                            "(hat lines concurrent on the side stream: in neither kind; no graph replay)"),
    }
    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "ms_per_step_median": statistics.median(step_ms), "ms_per_step_minmax": [min(step_ms), max(step_ms)],
        "config": {"workload": f"config{cfg.idx}:{cfg.name}", "N_x": Nx, "N_y": Ny, "J": J, "dofs": Nx * Ny,
                   "n": [cfg.nx, cfg.ny], "p": [cfg.px, cfg.py], "omega": cfg.omega,
                   "bc": "neumann" if cfg.bc else "dirichlet", "tol": cfg.tol, "mesh": cfg.mesh,
                   "step": "hpfem_load + hpfem_solve", "parallelism": f"replicas{ws}",
                   "l2_flush": ("not needed: every array exceeds the 126 MB L2" if 8.0 * Nx * Ny > 126e6 else
                                "none: arrays are L2-resident at this config (an L2 number)"),
                   "plan_ms": plan_ms},
        "dof_per_s": value * Nx * Ny,
        "hbm_alg_GBps": roofline["solve_alg_GBps"] * ws,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "roofline": roofline,
        "e2e": e2e,
    }
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, Fleg, J)
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_batched(args, cfg):
    """--batch B > 1 (NEXT-1): B independent right-hand sides per step through
    hpfem_load (per problem) + hpfem_solve_batched; the small configurations'
    throughput line.  One GPU (replicas under torchrun like the default)."""
    import torch
    import torch.distributed as dist

    import paper_2402_11299_b200 as hp
    import workloads as W

    import numpy as np

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    stream = torch.cuda.current_stream()
    B = args.batch
    xs, ys = cfg.breakpoints()
    Fleg = np.stack([W.f_leg(cfg, seed=b) for b in range(B)])
    Fh = torch.from_numpy(Fleg).pin_memory()
    plan = hp.Plan(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol)
    Nx, Ny, J = plan.Nx, plan.Ny, plan.J
    Fd = Fh.to(f"cuda:{dev}")
    Gd = torch.empty((B, Nx, Ny), dtype=torch.float64, device=dev)
    Ud = torch.empty_like(Gd)
    Uh = torch.empty((B, Nx, Ny), dtype=torch.float64).pin_memory()

    def step():
        for b in range(B):
            plan.load(Fd[b], Gd[b])
        plan.solve_batched(Gd, Ud)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_id_for(dev)) as clk:
        barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = plan.launches() + B  # the batched solve's kernels + one load per problem
    t_max_s = reduce_max(start.elapsed_time(end) / 1e3, f"cuda:{dev}" if ws > 1 else None)
    value = B * job_value(ws, args.steps, t_max_s)
    ms_per_step = t_max_s * 1e3 / args.steps
    e2e = None
    if not args.no_e2e:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            Fd.copy_(Fh, non_blocking=True)
            step()
            Uh.copy_(Ud, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        te = reduce_max(e0.elapsed_time(e1) / 1e3, f"cuda:{dev}" if ws > 1 else None)
        e2e = {"value": B * job_value(ws, args.steps, te), "unit": "solves/s",
               "h2d_bytes_per_step": int(Fh.numel() * 8), "d2h_bytes_per_step": int(Uh.numel() * 8),
               "ms_per_step": te * 1e3 / args.steps}
    peak, peak_kind = measured_peak()
    alg = 8.0 * Nx * Ny * (6 * J + 1) * B
    achieved = alg / (ms_per_step / 1e3) / 1e9
    resident = 3 * 8.0 * Nx * Ny * min(B, 8) < 126e6
    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{cfg.idx}:{cfg.name}", "batch": B, "N_x": Nx, "N_y": Ny, "J": J,
                   "step": f"{B} x hpfem_load + hpfem_solve_batched", "parallelism": f"replicas{ws}",
                   "l2_flush": ("none: the working set of the concurrent solves is L2-resident, "
                                "so this is an L2 throughput number") if resident else "not needed"},
        "dof_per_s": value * Nx * Ny,
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "kernel": "whole batched solve (algorithmic bytes 8 N_x N_y (6J+1) per problem)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)", "traffic": None},
        "e2e": e2e,
    }
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, Fleg[0], J)
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=5, choices=(1, 2, 3, 4, 5))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=1, help="B > 1: B right-hand sides per step (hpfem_solve_batched)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    import workloads as W

    cfg = W.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.batch > 1:
        return run_batched(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
