"""hpfem_apply (K7, F = A_x U M_y + M_x U A_y), hpfem_load (K8) and hpfem_unload (K9) timings against their
one-read-one-write rooflines:
    python scripts/bench_apply.py [CONFIG ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2402_11299_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402

try:
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    peak = 6650.0
for ci in [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]:
    c = W.CONFIGS[ci]
    xs, ys = c.breakpoints()
    plan = hp.Plan(xs, c.px, ys, c.py, c.omega, c.bc, c.tol)
    U = torch.randn(plan.Nx, plan.Ny, dtype=torch.float64, device="cuda")
    F = torch.empty_like(U)
    for _ in range(3):
        plan.apply(U, F)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        plan.apply(U, F)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gbs = 16.0 * plan.Nx * plan.Ny / (ms / 1e3) / 1e9
    res = {"config": ci, "N": [plan.Nx, plan.Ny], "apply_ms": ms, "dof_per_s": plan.Nx * plan.Ny / (ms / 1e3),
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                        "bytes_per_dof": 16}}
    # K8 load (G = R^T M_P F_leg M_P R) and K9 unload (C_leg = R U R^T): one read of the
    # source array + one write of the result
    nl, ml = (c.px + 1) * (len(xs) - 1), (c.py + 1) * (len(ys) - 1)
    Fl = torch.randn(nl, ml, dtype=torch.float64, device="cuda")
    Cl = torch.empty_like(Fl)
    for name, fn in (("load", lambda: plan.load(Fl, F)), ("unload", lambda: plan.unload(U, Cl))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
        by = 8.0 * (nl * ml + plan.Nx * plan.Ny)
        res[name + "_ms"] = t
        res[name + "_roofline"] = {"bound": "hbm", "achieved": by / (t / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                                   "frac": by / (t / 1e3) / 1e9 / peak, "bytes": by}
    print(json.dumps(res), flush=True)
    plan.close()
