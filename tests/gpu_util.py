"""Helpers for the GPU parity tests: run the CUDA path through the C ABI
binding and compare with the oracle in the Lemma 5.1 (L2) norm."""
from __future__ import annotations

import numpy as np

import oracle


def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        import pytest

        pytest.skip("no CUDA device")
    return torch


def gpu_plan(xs, px, ys, py, omega, bc, tol, robin=None):
    import paper_2402_11299_b200 as hp

    return hp.Plan(xs, px, ys, py, omega, bc, tol, robin=robin)


def gpu_solve(plan, G: np.ndarray, iters=None) -> np.ndarray:
    torch = torch_cuda()
    Gd = torch.from_numpy(np.ascontiguousarray(G)).cuda()
    Ud = torch.empty_like(Gd)
    plan.solve(Gd, Ud, iters=iters)
    torch.cuda.synchronize()
    return Ud.cpu().numpy()


def gpu_apply(plan, U: np.ndarray) -> np.ndarray:
    torch = torch_cuda()
    Ud = torch.from_numpy(np.ascontiguousarray(U)).cuda()
    Fd = torch.empty_like(Ud)
    plan.apply(Ud, Fd)
    torch.cuda.synchronize()
    return Fd.cpu().numpy()


def gpu_load(plan, Fleg: np.ndarray) -> np.ndarray:
    torch = torch_cuda()
    Fd = torch.from_numpy(np.ascontiguousarray(Fleg)).cuda()
    Gd = torch.empty((plan.Nx, plan.Ny), dtype=torch.float64, device="cuda")
    plan.load(Fd, Gd)
    torch.cuda.synchronize()
    return Gd.cpu().numpy()


def gpu_unload(plan, U: np.ndarray) -> np.ndarray:
    torch = torch_cuda()
    Ud = torch.from_numpy(np.ascontiguousarray(U)).cuda()
    Cd = torch.empty(((plan.px + 1) * plan.nx, (plan.py + 1) * plan.ny), dtype=torch.float64, device="cuda")
    plan.unload(Ud, Cd)
    torch.cuda.synchronize()
    return Cd.cpu().numpy()


def parity(xs, px, ys, py, bc, U, Uref):
    """(L2 relative, plain coefficient 2-norm relative, max-abs relative)
    differences (oracle.rel_diffs)."""
    return oracle.rel_diffs(xs, px, ys, py, bc, U, Uref)


# Floor of the element-sensitive measures on well-conditioned problems, where
# the perturbation floor itself can fall to a few ulps: 1e-14 ~ 45 u
# (u = 2^-53), a handful of roundings of differently ordered arithmetic.
ABS_REL_MIN = 1e-14


def floor_bound(floor, key, k=10.0, lo=ABS_REL_MIN):
    """k x the oracle's own rounding floor for measure `key` ("l2", "plain",
    "max"): the larger of its two perturbations (scripts/oracle_floor.py,
    oracle.rounding_floor), never below `lo`."""
    return max(lo, k * max(floor[f"G_perturb_{key}"], floor[f"mesh_ulp_{key}"]))


def assert_parity(tag, d, floor=None, l2_tol=1e-10, k=10.0):
    """d = parity(...).  L2 <= max(l2_tol, k x L2 floor) (north_star 1e-10,
    reading R12); with a floor also the plain-coefficient and max-abs
    differences <= k x their floors -- these weight the high-degree bubble
    coefficients as much as the hats, which the mass norm does not."""
    l2, plain, mx = d
    b_l2 = l2_tol if floor is None else max(l2_tol, k * max(floor["G_perturb_l2"], floor["mesh_ulp_l2"]))
    msg = f"{tag}: L2 {l2:.2e} (<= {b_l2:.1e}) plain {plain:.2e}"
    if floor is not None:
        b_p, b_m = floor_bound(floor, "plain", k), floor_bound(floor, "max", k)
        msg += f" (<= {b_p:.1e}) max {mx:.2e} (<= {b_m:.1e})"
    else:
        msg += f" max {mx:.2e}"
    print(msg)
    assert l2 <= b_l2, msg
    if floor is not None:
        assert plain <= b_p, msg
        assert mx <= b_m, msg


def golden_floor(key):
    """Recorded oracle floor (tests/golden/oracle_floor.json)."""
    import json
    import os

    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_floor.json")))[key]


def swapped_problem(xs, px, ys, py, bc, robin=None):
    """The transposed problem (x <-> y) of the same equation: arguments for
    the oracle when the plan solves A_y U^T M_x + M_y U^T A_x = G^T (reading
    R23, hpfem_plan_path reports it)."""
    bx, by = oracle.split_bc(bc)
    rob = None if robin is None else [robin[2], robin[3], robin[0], robin[1]]
    return ys, py, xs, px, oracle.bc2d(by, bx), rob


def oracle_reference(plan, xs, px, ys, py, om, bc, tol, G, iters=-1, floor=True):
    """(floor dict or None, Uref) from the oracle running Alg. 2 in the same
    orientation as the plan (the transposed equation when the plan is
    transposed; U returned in the caller's layout either way)."""
    tr = plan.path()["transposed"]
    if tr:
        xs, px, ys, py, bc, _ = swapped_problem(xs, px, ys, py, bc)
        G = np.ascontiguousarray(np.asarray(G).T)
    if floor:
        fl, U = oracle.rounding_floor(xs, px, ys, py, om, bc, tol, G, iters)
    else:
        fl, (U, _) = None, oracle.adi_solve(xs, px, ys, py, om, bc, tol, G, iters)
    return fl, (np.ascontiguousarray(U.T) if tr else U)
