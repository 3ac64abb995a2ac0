"""Diagnosis: config-5 load + a 1-iteration solve (load / copy-in / finalize kernels under ncu)."""
import sys, torch
sys.path.insert(0, "/root/repo")
import workloads, paper_2402_11299_b200 as hp
cfg = workloads.CONFIGS[5]
xs, ys = cfg.breakpoints()
plan = hp.Plan(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol)
Fl = torch.randn((cfg.px + 1) * len(xs[1:]), (cfg.py + 1) * len(ys[1:]), dtype=torch.float64, device="cuda")
G = torch.empty(plan.Nx, plan.Ny, dtype=torch.float64, device="cuda")
U = torch.empty_like(G)
plan.load(Fl, G)
plan.solve(G, U, iters=1)
torch.cuda.synchronize()
