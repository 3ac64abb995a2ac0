"""1D solver workload (NEXT-2 of SURVEY 8(f), the paper's Fig. 1: P:L618-L634):
time to plan/factor and to solve (K + w^2 M) u = f, Dirichlet, w = 1, for
several (n, p) at fixed N = n p - 1; a single right-hand side (latency) and a
batch of 1024 (throughput, HBM roofline: 16 algorithmic bytes per dof, F
read + U written, against MEASURED_PEAKS.json hbm_gbs).  Prints one JSON
line per shape and a summary line with the max/min time ratio over n at each
N (Fig. 1's claim: time roughly independent of n at fixed N)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_11299_b200 as hp  # noqa: E402


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def main():
    peak, src = peak_gbs()
    summary = {}
    for N0 in (1 << 12, 1 << 16):
        times = {}
        times1 = {}
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
                if nrhs > 1:
                    gbs = 16.0 * nrhs * N / (ms / 1e3) / 1e9
                    res["roofline"] = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                                       "frac": gbs / peak, "peak_source": src, "bytes_per_dof": 16}
                    times[n] = ms
                else:
                    times1[n] = ms
            pl.close()
            print(json.dumps(res), flush=True)
        summary[f"N={N0 - 1}"] = {"max_over_min_time_nrhs1024": max(times.values()) / min(times.values()),
                                  "max_over_min_time_nrhs1": max(times1.values()) / min(times1.values())}
    print(json.dumps({"summary": summary}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
