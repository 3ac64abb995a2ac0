"""Small solves on every kernel path, for compute-sanitizer (memcheck /
synccheck / racecheck / initcheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_cases.py

Covers K11 (config 1), the LDG half-step kernels (config 1 without K11), the
TMA ring kernels k_xstep_tma / k_ystep_tma with short (config 2, CL = 16)
and full-length chains (CL = 64, the config-5 kernel shape), the hat-line and
hat Schur kernels, load / unload / apply, the two-threads-per-chain x kernel
(natively and on the transposed path), the 1D solver (cluster form and
row-per-CTA form) and a batched solve.
Each result is checked against the oracle (L2 <= 1e-10), so a tool that
perturbs the run cannot pass silently.  HPFEM_NO_GRAPH=1: kernels are
launched directly (one sanitizer record per launch)."""
import os
import sys

os.environ["HPFEM_NO_GRAPH"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2402_11299_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402


def run(tag, xs, px, ys, py, om, bc, tol, env=None):
    for k in ("HPFEM_NO_SMALL", "HPFEM_NO_TMA"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    plan = hp.Plan(xs, px, ys, py, om, bc, tol)
    nx, ny = len(xs) - 1, len(ys) - 1
    Fleg = W.random_field(((px + 1) * nx, (py + 1) * ny), 1)
    Fd = torch.from_numpy(Fleg).cuda()
    G = torch.empty((plan.Nx, plan.Ny), dtype=torch.float64, device="cuda")
    U = torch.empty_like(G)
    plan.load(Fd, G)
    plan.solve(G, U)
    A = torch.empty_like(G)
    plan.apply(U, A)
    C = torch.empty_like(Fd)
    plan.unload(U, C)
    torch.cuda.synchronize()
    Gh = G.cpu().numpy()
    Uref, _ = oracle.adi_solve(xs, px, ys, py, om, bc, tol, Gh)
    l2 = oracle.l2_rel_diff(xs, px, ys, py, bc, U.cpu().numpy(), Uref)
    print(f"{tag}: N={plan.Nx}x{plan.Ny} J={plan.J} L2 {l2:.2e}", flush=True)
    assert l2 <= 1e-10
    plan.close()


c1, c2 = W.CONFIGS[1], W.CONFIGS[2]
x1, y1 = c1.breakpoints()
x2, y2 = c2.breakpoints()
run("config 1 K11", x1, c1.px, y1, c1.py, c1.omega, c1.bc, c1.tol)
run("config 1 LDG", x1, c1.px, y1, c1.py, c1.omega, c1.bc, c1.tol, {"HPFEM_NO_SMALL": "1"})
run("config 2 TMA CL=16", x2, c2.px, y2, c2.py, c2.omega, c2.bc, c2.tol)
g6, g5 = W.graded_mesh(0, 1, 6, 0.85), W.graded_mesh(0, 1, 5, 0.85)
run("graded p=128 Neumann TMA CL=64", g6, 128, g5, 128, 1.0, 1, 1e-10)
run("p=150 LDG long chains", np.linspace(0, 1, 3), 150, np.linspace(0, 1, 2), 140, 0.5, 0, 1e-8)
# round 2: chains of 65-128 positions with two threads per chain (k_xstep_tma2), natively and transposed
rng = np.random.default_rng(45)


def rmesh(n, a, b):
    w = rng.uniform(0.3, 1.7, size=n)
    xs = np.concatenate([[0.0], np.cumsum(w)])
    return a + (b - a) * xs / xs[-1]


run("p_x=130 two threads per x chain", rmesh(2, 0, 1), 130, rmesh(7, 0, 1), 18, 1.0, 1, 1e-10)
run("p_y=200 transposed, two threads per chain", rmesh(4, 0, 1), 20, rmesh(3, 0, 1), 200, 1.0, 0, 1e-10)
# 1D solver: cluster form (clusters of 1 and 2 CTAs), row-per-CTA form with two rows per CTA
for xs1, p1, nrhs, env in ((np.linspace(0, 1, 9), 8, 4, "1"), (np.linspace(0, 1, 513), 33, 3, "1"),
                           (np.linspace(0, 1, 41), 5, 601, "0")):
    os.environ["HPFEM_1D_CLUSTER"] = env
    pl = hp.Plan1D(xs1, p1, 0, 1.0)
    F = torch.randn((nrhs, pl.N), dtype=torch.float64, device="cuda")
    Uo = torch.empty_like(F)
    pl.solve(F, Uo)
    torch.cuda.synchronize()
    ref = oracle.solve1d(xs1, p1, 0, 1.0, 1.0, F.cpu().numpy())
    err = np.linalg.norm(Uo.cpu().numpy() - ref) / np.linalg.norm(ref)
    print(f"1D n={len(xs1) - 1} p={p1} rows={nrhs} cluster={env}: rel err {err:.2e}", flush=True)
    assert err <= 1e-10
    pl.close()
os.environ.pop("HPFEM_1D_CLUSTER", None)
# 1D solver and batched solve
pl = hp.Plan1D(np.linspace(0, 1, 9), 8, 0, 1.0)
F = torch.randn((4, pl.N), dtype=torch.float64, device="cuda")
Uo = torch.empty_like(F)
pl.solve(F, Uo)
torch.cuda.synchronize()
assert np.allclose(Uo.cpu().numpy(), oracle.solve1d(np.linspace(0, 1, 9), 8, 0, 1.0, 1.0, F.cpu().numpy()), rtol=1e-10,
                   atol=1e-12)
pl.close()
plan = hp.Plan(x2, c2.px, y2, c2.py, c2.omega, c2.bc, c2.tol)
Fb = torch.randn((3, plan.Nx, plan.Ny), dtype=torch.float64, device="cuda")
Ub = torch.empty_like(Fb)
plan.solve_batched(Fb, Ub)
torch.cuda.synchronize()
plan.close()
print("sanitize cases: all ok", flush=True)
