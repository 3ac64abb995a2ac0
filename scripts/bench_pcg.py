"""NEXT-3 workload (Section 7, Table 1): hpfem_pcg on the
singular variable-coefficient problem (-Delta - 10 log r) u = 1 on (-1,1)^2
with the graded mesh T_m, ADI preconditioner tolerance 1e-4, CG relative
tolerance 1e-8.  Inputs come from the product path only (grid from
hpfem_grid, f = 1 loaded by hpfem_load).  Per (m, p): PCG solves/s,
iterations, and the time split into the ADI preconditioner, the
variable-coefficient operator and its transform passes; the transform
kernel's fp64 flop rate is reported against the measured FP64 FMA peak
(scripts/micro/dfma_peak.cu) when --fp64-peak is given.  One JSON line per
shape."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_11299_b200 as hp  # noqa: E402


def graded(m):
    pos = [10.0 ** (-j) for j in range(m, 0, -1)]
    return np.array([-1.0] + [-v for v in reversed(pos)] + [0.0] + pos + [1.0])


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(m, p, reps, fp64_peak):
    xs = graded(m)
    n = xs.size - 1
    s = torch.cuda.current_stream().cuda_stream
    plan = hp.Plan(xs, p, xs, p, 0.0, hp.HPFEM_BC_DIRICHLET, 1e-4, stream=s)
    gx, gy = plan.grid()
    cg = torch.from_numpy(-10.0 * np.log(np.sqrt(gx[:, None] ** 2 + gy[None, :] ** 2))).cuda()
    L = (p + 1) * n
    Fleg = torch.zeros((L, L), dtype=torch.float64, device="cuda")
    Fleg[:n, :n] = 1.0
    G = torch.empty((plan.Nx, plan.Ny), dtype=torch.float64, device="cuda")
    plan.load(Fleg, G, stream=s)
    U = torch.empty_like(G)
    out = {}
    out["pcg_ms"] = timed(lambda: out.update(zip(("iters", "relres"), plan.pcg(cg, G, U, 1e-8, 200, stream=s))),
                          reps)
    Z = torch.empty_like(G)
    out["adi_ms"] = timed(lambda: plan.solve(G, Z, stream=s), reps)
    out["varcoef_ms"] = timed(lambda: plan.varcoef_apply(cg, G, Z, stream=s), reps)
    C = torch.empty((L, L), dtype=torch.float64, device="cuda")
    out["transform_ms"] = timed(lambda: plan.transform(cg, C, stream=s), reps)
    flops = 2.0 * 2 * (p + 1) * L * L  # two passes, (p+1) FMAs per output
    out["transform_tflops"] = flops / (out["transform_ms"] * 1e-3) / 1e12
    if fp64_peak:
        out["transform_frac_of_fp64_peak"] = out["transform_tflops"] / fp64_peak
    res = {"workload": f"table1_m{m}_p{p}", "cells": n * n, "N": plan.Nx, "J_pre": plan.J,
           "pcg_solves_per_s": 1e3 / out["pcg_ms"], "dof_per_s": plan.Nx * plan.Ny * 1e3 / out["pcg_ms"], **out}
    plan.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fp64-peak", type=float, default=0.0, help="measured FP64 FMA TFLOP/s")
    ap.add_argument("--shapes", default="1:8,1:32,2:64,3:64,3:128")
    a = ap.parse_args()
    for sh in a.shapes.split(","):
        m, p = map(int, sh.split(":"))
        print(json.dumps(run(m, p, a.reps, a.fp64_peak)), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
