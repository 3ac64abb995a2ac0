"""NEXT-4 workload (Section 6, Fig. 'burgers' P:L955-L985): time per IMEX
step of u_t + u u_x = eps Delta u on (-1,1)^2, zero Dirichlet data, eps = 0.1
(Fig. caption), piecewise-constant random initial data on the 9 x 9 element
grid of Fig. 'discont' (refined by an integer factor for the large shapes),
dt = 1e-3, ADI tolerance 1e-10.  Inputs built on the device (Legendre
coefficients: degree 0 = the cell value).  Per shape: ms per step, DOF/s,
and the split into the ADI solve and the transform / nonlinear part.  One
JSON line per shape."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_11299_b200 as hp  # noqa: E402


def run(n, p, steps, eps=0.1, dt=1e-3, tol=1e-10):
    xs = np.linspace(-1.0, 1.0, n + 1)
    s = torch.cuda.current_stream().cuda_stream
    plan = hp.Plan(xs, p, xs, p, 1.0 / np.sqrt(dt * eps), hp.HPFEM_BC_DIRICHLET, tol, stream=s)
    L = (p + 1) * n
    U = torch.zeros((L, L), dtype=torch.float64, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    U[:n, :n] = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    V = torch.empty_like(U)
    for _ in range(2):
        plan.imex_step(dt, U, V, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(steps):
        plan.imex_step(dt, U, V, stream=s) if k % 2 == 0 else plan.imex_step(dt, V, U, stream=s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    G = torch.empty((plan.Nx, plan.Ny), dtype=torch.float64, device="cuda")
    W = torch.empty_like(G)
    plan.load(U, G, stream=s)
    e0.record()
    for _ in range(steps):
        plan.solve(G, W, stream=s)
    e1.record()
    torch.cuda.synchronize()
    adi = e0.elapsed_time(e1) / steps
    res = {"workload": f"burgers_n{n}_p{p}", "N": plan.Nx, "J": plan.J, "ms_per_step": ms,
           "steps_per_s": 1e3 / ms, "dof_per_s": plan.Nx * plan.Ny * 1e3 / ms, "adi_ms": adi,
           "nonlinear_ms": ms - adi}
    plan.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--shapes", default="9:8,9:16,9:32,9:64,9:128,36:128,72:64")
    a = ap.parse_args()
    for sh in a.shapes.split(","):
        n, p = map(int, sh.split(":"))
        print(json.dumps(run(n, p, a.steps)), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
