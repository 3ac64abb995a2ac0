"""Diagnosis: one config-5 solve with 3 ADI iterations (library built with -DHPFEM_YPROF prints per-warp cycle splits)."""
import sys, torch
sys.path.insert(0, "/root/repo")
import workloads, paper_2402_11299_b200 as hp
cfg = workloads.CONFIGS[5]
xs, ys = cfg.breakpoints()
plan = hp.Plan(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol)
G = torch.randn(plan.Nx, plan.Ny, dtype=torch.float64, device="cuda")
U = torch.empty_like(G)
plan.solve(G, U, iters=3)
torch.cuda.synchronize()
