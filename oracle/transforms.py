"""Oracle for NEXT-3 of SURVEY 8(f): grid <-> piecewise-Legendre transforms
(Section 6), the variable-coefficient operator of eq.
(evaluation) and ADI-preconditioned conjugate gradients
(Section 7).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy, fp64, no
blocking or fusion; the Legendre Vandermonde matrix comes from numpy
(`legvander`, a library primitive) and its inverse from LAPACK.  Readings of
the paper (R17-R20):
  R17  degree-p coefficients need p + 1 points: the paper's "p Chebyshev
       points" x_k = sin(pi (p - 2k + 1)/(2p)) are taken with
       m = p + 1 points, x_k = sin(pi (m - 2k + 1)/(2m)), k = 1..m (descending);
  R18  grid values are stored like the coefficients:
       row i*n + e = point i of element e (point-major, element-minor);
  R19  eq. (evaluation) prints R^{-1} M_P ... M_P R^{-T}; R is rectangular,
       and <v, g u> for v in the hat/bubble basis is the load R^T M_P (.) M_P R
       (P:L417), so the operator is
       F = R_x^T M_P F_x [G o (F_x^{-1} R_x U R_y^T F_y^{-T})] F_y^T M_P R_y;
  R20  CG stops when ||r_k||_2 <= rtol ||b||_2 (x_0 = 0), Saad's PCG.
"""
from __future__ import annotations

import numpy as np


def cheb_points(m: int) -> np.ndarray:
    """m Chebyshev points of the first kind, x_k = sin(pi (m - 2k + 1)/(2m)),
    k = 1..m, descending."""
    k = np.arange(1, m + 1)
    return np.sin(np.pi * (m - 2 * k + 1) / (2 * m))


def grid_1d(xs, p: int) -> np.ndarray:
    """Points of the 1D grid, affine images of cheb_points(p + 1) on every
    element (P:L917 'affine transform the grid'), point-major / element-minor
    (reading R18): g[i n + e]."""
    xs = np.asarray(xs, dtype=np.float64)
    n = xs.size - 1
    t = cheb_points(p + 1)
    g = np.empty((p + 1) * n)
    for i in range(p + 1):
        for e in range(n):
            g[i * n + e] = xs[e] + (t[i] + 1.0) * (xs[e + 1] - xs[e]) / 2.0
    return g


def vandermonde(p: int) -> np.ndarray:
    """V[i, k] = P_k(x_i) on the reference points: the inverse transform
    F_p^{-1} (Legendre coefficients -> values)."""
    return np.polynomial.legendre.legvander(cheb_points(p + 1), p)


def transform_matrix(p: int) -> np.ndarray:
    """F_p = V^{-1}: values at the p + 1 points -> Legendre coefficients of
    the degree-p interpolant (c = F_p f(x))."""
    return np.linalg.inv(vandermonde(p))


def _apply_blocks(A: np.ndarray, X: np.ndarray, n: int, axis: int) -> np.ndarray:
    """Apply the per-element matrix A to every element block of axis `axis`
    (index i n + e -> k n + e)."""
    X = np.asarray(X, dtype=np.float64)
    if axis == 0:
        Xb = X.reshape(A.shape[1], n, X.shape[1])
        return np.einsum("ki,iej->kej", A, Xb).reshape(A.shape[0] * n, X.shape[1])
    Xb = X.reshape(X.shape[0], A.shape[1], n)
    return np.einsum("ki,rie->rke", A, Xb).reshape(X.shape[0], A.shape[0] * n)


def transform(px: int, nx: int, py: int, ny: int, Vals) -> np.ndarray:
    """2D transform F_p^n F (F_q^m)^T: grid values -> piecewise
    Legendre coefficients (degree-major / element-minor in both dimensions)."""
    C = _apply_blocks(transform_matrix(px), Vals, nx, 0)
    return _apply_blocks(transform_matrix(py), C, ny, 1)


def itransform(px: int, nx: int, py: int, ny: int, C) -> np.ndarray:
    """Inverse 2D transform (F_p^n)^{-1} C (F_q^m)^{-T}:
    piecewise Legendre coefficients -> grid values."""
    V = _apply_blocks(vandermonde(px), C, nx, 0)
    return _apply_blocks(vandermonde(py), V, ny, 1)


def coefficient_grid(xs, px, ys, py, fun) -> np.ndarray:
    """G = [g(x_k, y_j)] on the tensor grid."""
    gx, gy = grid_1d(xs, px), grid_1d(ys, py)
    return np.array(np.broadcast_to(fun(gx[:, None], gy[None, :]), (gx.size, gy.size)), dtype=np.float64)


def varcoef_apply(xs, px, ys, py, bc, cgrid, U, omega=0.0) -> np.ndarray:
    """(A_x (x) M_y + M_x (x) A_y) U + <v, c u>, A = K + (w^2/2) M (w = 0 in
    Section 7: the weak Laplacian), with <v, c u> evaluated by eq.
    (evaluation) (reading R19):
        R_x^T M_P F_x [c o (F_x^{-1} R_x U R_y^T F_y^{-T})] F_y^T M_P R_y."""
    from . import apply, load, unload

    xs, ys = np.asarray(xs, dtype=np.float64), np.asarray(ys, dtype=np.float64)
    nx, ny = xs.size - 1, ys.size - 1
    C = unload(xs, px, ys, py, bc, U)                  # R_x U R_y^T
    V = itransform(px, nx, py, ny, C)                  # values on the grid
    Cg = transform(px, nx, py, ny, np.asarray(cgrid) * V)  # Legendre coefficients of I(c u)
    return apply(xs, px, ys, py, omega, bc, U) + load(xs, px, ys, py, bc, Cg)


def pcg(xs, px, ys, py, bc, cgrid, b, rtol=1e-8, maxit=200, tol_pre=1e-4, omega=0.0):
    """Preconditioned conjugate gradients (Saad, Alg. 9.1) for the operator of
    varcoef_apply, preconditioned by the ADI solve of the weak Laplacian
    (screened by w if w != 0) with tolerance tol_pre (Table 1
    P:L1039).  x_0 = 0;
    stops when ||r_k||_2 <= rtol ||b||_2 (reading R20).  Returns
    (U, iterations, relative residual history)."""
    from . import adi_solve

    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    nb = float(np.linalg.norm(b))
    hist = [1.0]
    if nb == 0.0:
        return x, 0, hist
    z, _ = adi_solve(xs, px, ys, py, omega, bc, tol_pre, r)
    p = z.copy()
    rz = float(np.sum(r * z))
    it = 0
    while it < maxit:
        q = varcoef_apply(xs, px, ys, py, bc, cgrid, p, omega)
        alpha = rz / float(np.sum(p * q))
        x = x + alpha * p
        r = r - alpha * q
        it += 1
        hist.append(float(np.linalg.norm(r)) / nb)
        if hist[-1] <= rtol:
            break
        z, _ = adi_solve(xs, px, ys, py, omega, bc, tol_pre, r)
        rz_new = float(np.sum(r * z))
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it, hist


def graded_mesh_Tm(m: int) -> np.ndarray:
    """Cell end points (-1, -10^{-1}, ..., -10^{-m}, 0, 10^{-m}, ..., 10^{-1}, 1)
    of eq. (graded-mesh)."""
    pos = [10.0 ** (-j) for j in range(m, 0, -1)]
    return np.array([-1.0] + [-v for v in reversed(pos)] + [0.0] + pos + [1.0])


# ------------------------------------------------------------------ NEXT-4
def unload_matrix_1d(xs, p: int, bc: int) -> np.ndarray:
    """Dense R ((p+1) n x N): Legendre coefficients of the hat/bubble
    expansion, W_k = (P_k - P_{k+2})/(2k+3) (eq. app:1), hats
    (1 -+ t)/2 = P_0/2 -+ P_1/2."""
    from . import dim

    xs = np.asarray(xs, dtype=np.float64)
    n = xs.size - 1
    N = dim(n, p, bc)
    dl, dr = bc in (0, 2), bc in (0, 3)
    nh = n + 1 - dl - dr
    R = np.zeros(((p + 1) * n, N))
    for e in range(n):
        for side, node in ((0, e), (1, e + 1)):
            if (node == 0 and dl) or (node == n and dr):
                continue
            h = node - (1 if dl else 0)
            R[e, h] += 0.5
            R[n + e, h] += -0.5 if side == 0 else 0.5
        for k in range(p - 1):
            R[k * n + e, nh + k * n + e] += 1.0 / (2 * k + 3)
            R[(k + 2) * n + e, nh + k * n + e] += -1.0 / (2 * k + 3)
    return R


def deriv_matrix_1d(xs, p: int, bc: int) -> np.ndarray:
    """Dense D ((p+1) n x N): Legendre coefficients of du/dx.  On an element
    of width delta, dx = (delta/2) dt, W_k' = -P_{k+1} and the hats
    (1 -+ t)/2 have slopes -+ 1/delta."""
    from . import dim

    xs = np.asarray(xs, dtype=np.float64)
    n = xs.size - 1
    N = dim(n, p, bc)
    dl, dr = bc in (0, 2), bc in (0, 3)
    nh = n + 1 - dl - dr
    D = np.zeros(((p + 1) * n, N))
    for e in range(n):
        d = xs[e + 1] - xs[e]
        for side, node in ((0, e), (1, e + 1)):
            if (node == 0 and dl) or (node == n and dr):
                continue
            D[e, node - (1 if dl else 0)] += (-1.0 if side == 0 else 1.0) / d
        for k in range(p - 1):
            D[(k + 1) * n + e, nh + k * n + e] += -2.0 / d
    return D


def deriv_unload(xs, px, ys, py, bc, U) -> np.ndarray:
    """Legendre coefficients of du/dx: D_x U R_y^T."""
    from . import split_bc

    bx, by = split_bc(bc)
    return deriv_matrix_1d(xs, px, bx) @ np.asarray(U, dtype=np.float64) @ unload_matrix_1d(ys, py, by).T


def explicit_step(xs, px, ys, py, dt, W) -> np.ndarray:
    """Nonlinear half-step of the IMEX scheme on the
    grid: U_{k+1} = F [V - dt V_x o V] with V = F^{-1} R W R^T F^{-T} and
    V_x = F^{-1} D W R^T F^{-T}.  The sign is that of the PDE
    u_t + u u_x = eps Delta u (the listing prints '+', reading
    R21).  Zero Dirichlet ends."""
    from . import unload

    xs, ys = np.asarray(xs, dtype=np.float64), np.asarray(ys, dtype=np.float64)
    nx, ny = xs.size - 1, ys.size - 1
    V = itransform(px, nx, py, ny, unload(xs, px, ys, py, 0, W))
    Vx = itransform(px, nx, py, ny, deriv_unload(xs, px, ys, py, 0, W))
    return transform(px, nx, py, ny, V - dt * (Vx * V))


def imex_step(xs, px, ys, py, eps, dt, tol, Uleg) -> np.ndarray:
    """One step of u_t + u u_x = eps Delta u, zero Dirichlet:
    implicit Euler u_{k+1/2} = (I - dt eps Delta)^{-1} u_k as the screened
    problem (K(x)M + M(x)K + w^2 M(x)M) W = w^2 <v, u_k>, w = 1/sqrt(dt eps),
    by ADI (Alg. 2), then explicit_step.  Uleg: piecewise Legendre
    coefficients (the F_leg layout)."""
    from . import adi_solve, load

    w = 1.0 / np.sqrt(dt * eps)
    G = load(xs, px, ys, py, 0, Uleg) * (w * w)
    W, _ = adi_solve(xs, px, ys, py, w, 0, tol, G)
    return explicit_step(xs, px, ys, py, dt, W)


def legendre_l2_sq(xs, px, ys, py, C) -> float:
    """||u||^2_{L2} of a piecewise tensor Legendre expansion (||P_k||^2 =
    2/(2k+1), scaled by delta/2 per direction)."""
    xs, ys = np.asarray(xs, dtype=np.float64), np.asarray(ys, dtype=np.float64)
    nx, ny = xs.size - 1, ys.size - 1
    wx = np.array([(xs[e + 1] - xs[e]) / (2 * k + 1) for k in range(px + 1) for e in range(nx)])
    wy = np.array([(ys[e + 1] - ys[e]) / (2 * k + 1) for k in range(py + 1) for e in range(ny)])
    return float(np.einsum("i,j,ij->", wx, wy, np.asarray(C) ** 2))
