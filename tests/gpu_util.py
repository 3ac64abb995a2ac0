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
    """(L2 relative difference, plain coefficient 2-norm relative difference)."""
    l2 = oracle.l2_rel_diff(xs, px, ys, py, bc, U, Uref)
    plain = float(np.linalg.norm(U - Uref) / np.linalg.norm(Uref)) if np.any(Uref) else float(np.linalg.norm(U))
    return l2, plain
