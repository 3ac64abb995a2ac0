"""Host-side submission time vs device time of one solve (launch-gap check)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2402_11299_b200 as hp, workloads as W
cfg = W.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
xs, ys = cfg.breakpoints()
plan = hp.Plan(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol)
G = torch.randn(plan.Nx, plan.Ny, dtype=torch.float64, device="cuda")
U = torch.empty_like(G)
for _ in range(2):
    plan.solve(G, U)
torch.cuda.synchronize()
for it in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter(); e0.record()
    plan.solve(G, U)
    t1 = time.perf_counter(); e1.record()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"host submit {1e3*(t1-t0):.1f} ms, device {e0.elapsed_time(e1):.1f} ms, wall {1e3*(t2-t0):.1f} ms, launches {plan.launches()}")
