"""One load + solve of a configuration (for ncu captures of single kernels):
    python scripts/prof_solve.py CONFIG [ITERS]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2402_11299_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

c = W.CONFIGS[int(sys.argv[1])]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else None
xs, ys = c.breakpoints()
plan = hp.Plan(xs, c.px, ys, c.py, c.omega, c.bc, c.tol)
F = torch.from_numpy(W.f_leg(c, seed=0)).cuda()
G = torch.empty((plan.Nx, plan.Ny), dtype=torch.float64, device="cuda")
U = torch.empty_like(G)
plan.load(F, G)
for _ in range(2):
    plan.solve(G, U, iters=iters)
torch.cuda.synchronize()
print("ok", plan.Nx, plan.Ny, plan.J, float(U.abs().max()))
