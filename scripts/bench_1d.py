"""1D solver workload (NEXT-2 of SURVEY 8(f), the paper's Fig. 1: P:L618-L634):
time to plan/factor and to solve (K + w^2 M) u = f, Dirichlet, w = 1, for
several (n, p) at fixed N = n p - 1; single right-hand side (latency) and a
batch of right-hand sides (throughput).  Prints one JSON line per shape."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2402_11299_b200 as hp  # noqa: E402


def main():
    out = []
    for N0 in (1 << 12, 1 << 16):
        for p in (4, 16, 64, 256):
            n = max(1, N0 // p)
            xs = np.linspace(-1.0, 1.0, n + 1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pl = hp.Plan1D(xs, p, 0, 1.0)
            t_plan = time.perf_counter() - t0
            N = pl.N
            res = {"n": n, "p": p, "N": N, "plan_ms": t_plan * 1e3}
            for nrhs in (1, 1024):
                F = torch.randn(nrhs, N, dtype=torch.float64, device="cuda")
                U = torch.empty_like(F)
                for _ in range(3):
                    pl.solve(F, U)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 20
                e0.record()
                for _ in range(reps):
                    pl.solve(F, U)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                res[f"solve_ms_nrhs{nrhs}"] = ms
                res[f"dof_per_s_nrhs{nrhs}"] = nrhs * N / (ms / 1e3)
            pl.close()
            out.append(res)
            print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
