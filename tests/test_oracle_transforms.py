"""Pins of the NEXT-3 oracle (oracle/transforms.py): grid <-> Legendre
transforms (Section 6), the variable-coefficient operator of
eq. (evaluation) and ADI-preconditioned CG (Section 7).

Pinned against library routines on special cases (numpy's Chebyshev points
and Legendre evaluation), exactness on polynomials, the mass-matrix special
case c = const, an exact polynomial solution, and the iteration counts the
paper prints in Table 1 (tests/golden/table1_pcg_iters.json).  CPU only.
"""
import json
import os

import numpy as np
import pytest
from numpy.polynomial import legendre as npleg

import oracle
from oracle import transforms as T

RNG = np.random.default_rng(77)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1_pcg_iters.json")


def rand_mesh(n, a=-1.0, b=1.0, seed=0):
    w = np.random.default_rng(seed).uniform(0.3, 1.7, size=n)
    xs = np.concatenate([[0.0], np.cumsum(w)])
    return a + (b - a) * xs / xs[-1]


@pytest.mark.parametrize("m", [1, 2, 5, 9, 33])
def test_cheb_points_are_first_kind(m):
    """the points are the first-kind Chebyshev points (numpy's
    chebpts1, ascending), listed in descending order."""
    x = T.cheb_points(m)
    assert np.all(np.diff(x) < 0) or m == 1
    np.testing.assert_allclose(x[::-1], np.polynomial.chebyshev.chebpts1(m), atol=2e-16)


@pytest.mark.parametrize("p", [2, 5, 8, 17, 32])
def test_transform_1d_exact_on_polynomials(p):
    """c = F_p f(x) recovers the Legendre coefficients of any
    polynomial of degree <= p (numpy legval evaluates it)."""
    c = RNG.standard_normal(p + 1)
    vals = npleg.legval(T.cheb_points(p + 1), c)
    np.testing.assert_allclose(T.transform_matrix(p) @ vals, c, atol=1e-13 * max(1, p))


def _eval_2d(xs, px, ys, py, C, x, y):
    """Direct evaluation of the piecewise Legendre expansion C (degree-major /
    element-minor) at a point, by numpy's legval2d on the element."""
    nx, ny = xs.size - 1, ys.size - 1
    ex = min(np.searchsorted(xs, x, side="right") - 1, nx - 1)
    ey = min(np.searchsorted(ys, y, side="right") - 1, ny - 1)
    tx = 2 * (x - xs[ex]) / (xs[ex + 1] - xs[ex]) - 1
    ty = 2 * (y - ys[ey]) / (ys[ey + 1] - ys[ey]) - 1
    Ce = C[ex::nx, :][:, ey::ny]
    return npleg.legval2d(tx, ty, Ce)


def test_itransform_2d_is_pointwise_evaluation():
    """(F_p^n)^{-1} C (F_q^m)^{-T} = the values of the piecewise
    expansion at the grid (checked point by point, independent evaluation),
    and the grid is the affine image of the points on every element."""
    xs, ys = rand_mesh(3, seed=1), rand_mesh(4, 0, 2, seed=2)
    px, py = 6, 5
    C = RNG.standard_normal(((px + 1) * 3, (py + 1) * 4))
    V = T.itransform(px, 3, py, 4, C)
    gx, gy = T.grid_1d(xs, px), T.grid_1d(ys, py)
    for i in range(0, gx.size, 2):
        for j in range(0, gy.size, 3):
            assert abs(V[i, j] - _eval_2d(xs, px, ys, py, C, gx[i], gy[j])) <= 1e-12 * np.abs(C).sum()
    # element e of the grid holds points in [x_e, x_{e+1}]
    for e in range(3):
        pts = gx[e::3]
        assert np.all(pts > xs[e]) and np.all(pts < xs[e + 1])
    np.testing.assert_allclose(T.transform(px, 3, py, 4, V), C, atol=1e-12)


def test_transform_converges_to_legendre_projection():
    """For a smooth function the interpolant's Legendre coefficients converge
    exponentially to the L2 projection's (Gauss quadrature, numpy leggauss)."""
    f = lambda x: np.exp(np.sin(2 * x))
    xs = np.array([-1.0, 0.3, 1.0])
    p = 30
    vals = f(T.grid_1d(xs, p))
    C = T._apply_blocks(T.transform_matrix(p), vals[:, None], 2, 0)[:, 0]
    tq, wq = npleg.leggauss(80)
    for e in range(2):
        x = xs[e] + (tq + 1) * (xs[e + 1] - xs[e]) / 2
        for k in range(12):
            ck = (2 * k + 1) / 2 * np.sum(wq * npleg.legval(tq, np.eye(k + 1)[k]) * f(x))
            assert abs(C[k * 2 + e] - ck) <= 1e-13


@pytest.mark.parametrize("bc,om", [(0, 0.0), (oracle.bc2d(2, 3), 0.0), (oracle.bc2d(2, 1), 1.5)])
def test_varcoef_constant_coefficient_is_mass(bc, om):
    """c = s constant: <v, s u> is exact (c u has degree p), so the operator is
    K_x(x)M_y + M_x(x)K_y + s M_x(x)M_y = the screened operator with w^2 = s
    (eq. 2d:poisson); with a screening w the total is w^2 + s."""
    xs, ys = rand_mesh(3, seed=3), rand_mesh(2, 0, 1, seed=4)
    px, py, s = 5, 7, 2.5
    Nx, Ny = oracle.dim(3, px, oracle.split_bc(bc)[0]), oracle.dim(2, py, oracle.split_bc(bc)[1])
    U = RNG.standard_normal((Nx, Ny))
    cg = T.coefficient_grid(xs, px, ys, py, lambda x, y: s + 0 * x * y)
    F = T.varcoef_apply(xs, px, ys, py, bc, cg, U, om)
    Fref = oracle.apply(xs, px, ys, py, np.sqrt(om * om + s), bc, U)
    np.testing.assert_allclose(F, Fref, atol=1e-12 * np.abs(Fref).max())


def test_pcg_exact_polynomial_solution():
    """u* = (1 - x^2)(1 - y^2) lies in the discrete space for p >= 2; with the
    polynomial coefficient c = 2 + x y^2 the interpolation of c u is exact for
    p >= 4 and f = -Delta u* + c u* (degree <= 7) is loaded exactly for
    p >= 7, so the Galerkin solution IS u*: PCG must return its coefficients
    (compared through the Legendre coefficients of u*)."""
    xs = rand_mesh(3, seed=5)
    ys = rand_mesh(2, seed=6)
    p = 8
    f = lambda x, y: 2 * (1 - y * y) + 2 * (1 - x * x) + (2 + x * y * y) * (1 - x * x) * (1 - y * y)
    Fleg = T.transform(p, 3, p, 2, T.coefficient_grid(xs, p, ys, p, f))
    b = oracle.load(xs, p, ys, p, 0, Fleg)
    cg = T.coefficient_grid(xs, p, ys, p, lambda x, y: 2 + x * y * y)
    U, it, hist = T.pcg(xs, p, ys, p, 0, cg, b, rtol=1e-13, maxit=60)
    C = oracle.unload(xs, p, ys, p, 0, U)
    Cstar = T.transform(p, 3, p, 2, T.coefficient_grid(xs, p, ys, p, lambda x, y: (1 - x * x) * (1 - y * y)))
    assert hist[-1] <= 1e-13 and it <= 20
    np.testing.assert_allclose(C, Cstar, atol=1e-11)


def test_graded_mesh_cells():
    """eq. (graded-mesh): 2(m + 1) cells per direction, i.e. the
    16 / 36 / 64 cells of Table 1."""
    g = json.load(open(GOLDEN))
    for m, cells in g["cells"].items():
        xs = T.graded_mesh_Tm(int(m))
        assert (xs.size - 1) ** 2 == cells and xs[0] == -1 and xs[-1] == 1
        assert np.all(np.diff(xs) > 0) and 0.0 in xs and 10.0 ** (-int(m)) in xs


def table1_problem(m, p):
    """eq. (variable-coeff) P:L999-L1002 on T_m: f = 1, c = -10 log r."""
    xs = T.graded_mesh_Tm(m)
    n = xs.size - 1
    Fleg = np.zeros(((p + 1) * n, (p + 1) * n))
    Fleg[:n, :n] = 1.0  # f = 1: the degree-0 coefficient on every element
    b = oracle.load(xs, p, xs, p, 0, Fleg)
    cg = T.coefficient_grid(xs, p, xs, p, lambda x, y: -10.0 * np.log(np.sqrt(x * x + y * y)))
    return xs, b, cg


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("p", [8, 16, 32, 64, 128])
def test_table1_iteration_counts(m, p):
    """The paper's printed PCG iteration counts (Table 1)."""
    g = json.load(open(GOLDEN))
    xs, b, cg = table1_problem(m, p)
    U, it, hist = T.pcg(xs, p, xs, p, 0, cg, b, rtol=g["rtol"], tol_pre=g["adi_tol"])
    assert it == g["iters"][str(m)][str(p)], (m, p, it, hist)


# ------------------------------------------------------------------ NEXT-4
@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_unload_matrix_matches_oracle_unload(bc):
    """The dense 1D R of the IMEX oracle equals the C++ oracle's unload
    (itself pinned against the Jacobi-defined basis)."""
    xs = rand_mesh(4, seed=bc)
    p = 6
    N = oracle.dim(4, p, bc)
    U = RNG.standard_normal((N, 1))
    ys = np.array([-1.0, 1.0])
    R = T.unload_matrix_1d(xs, p, bc)
    C = oracle.unload(xs, p, ys, 2, oracle.bc2d(bc, 0), np.hstack([U]))  # y: one Dirichlet element, one bubble
    np.testing.assert_allclose(R @ U[:, 0] * (1.0 / 3.0), C[:, 0], atol=1e-14)


def test_derivative_unload_is_legder():
    """D_x U R_y^T = the per-element Legendre derivative
    (numpy legder, times 2/delta) of the unloaded expansion."""
    xs, ys = rand_mesh(3, seed=11), rand_mesh(2, 0, 1, seed=12)
    px, py = 7, 5
    U = RNG.standard_normal((oracle.dim(3, px, 0), oracle.dim(2, py, 0)))
    C = oracle.unload(xs, px, ys, py, 0, U)
    Cx = T.deriv_unload(xs, px, ys, py, 0, U)
    for e in range(3):
        ref = npleg.legder(C[e::3, :], axis=0) * 2.0 / (xs[e + 1] - xs[e])
        np.testing.assert_allclose(Cx[e::3, :][:px], ref, atol=1e-12 * np.abs(ref).max())
        assert np.all(Cx[px * 3 + e, :] == 0.0)


def test_explicit_step_pointwise():
    """itransform(explicit_step(W)) = u - dt u u_x at every grid point, with u
    and u_x evaluated directly (numpy legval2d / legder on each element)."""
    xs, ys = rand_mesh(2, seed=13), rand_mesh(3, seed=14)
    px, py, dt = 6, 5, 0.05
    W = RNG.standard_normal((oracle.dim(2, px, 0), oracle.dim(3, py, 0)))
    Y = T.itransform(px, 2, py, 3, T.explicit_step(xs, px, ys, py, dt, W))
    C = oracle.unload(xs, px, ys, py, 0, W)
    gx, gy = T.grid_1d(xs, px), T.grid_1d(ys, py)
    for i in range(0, gx.size, 2):
        for j in range(0, gy.size, 2):
            u = _eval_2d(xs, px, ys, py, C, gx[i], gy[j])
            ex = min(np.searchsorted(xs, gx[i], side="right") - 1, 1)
            Cd = np.zeros_like(C)
            for e in range(2):
                Cd[e::2, :][:px] = npleg.legder(C[e::2, :], axis=0) * 2.0 / (xs[e + 1] - xs[e])
            ux = _eval_2d(xs, px, ys, py, Cd, gx[i], gy[j])
            assert abs(Y[i, j] - (u - dt * u * ux)) <= 1e-11 * (1 + abs(u) * (1 + abs(ux))), (i, j, ex)


def test_imex_linear_limit_heat_decay():
    """Amplitude 1e-10: the nonlinear term is dt |u_x| ~ 3e-12 relative, so one step
    is implicit Euler for the heat equation, whose exact action on the
    eigenfunction sin(pi x) sin(pi y) of (-1,1)^2 is division by
    1 + 2 pi^2 dt eps; p = 16 resolves it to ~1e-12."""
    xs = ys = np.linspace(-1, 1, 3)
    p, eps, dt, a = 16, 0.1, 0.01, 1e-10
    u0 = lambda x, y: a * np.sin(np.pi * x) * np.sin(np.pi * y)
    U0 = T.transform(p, 2, p, 2, T.coefficient_grid(xs, p, ys, p, u0))
    U1 = T.imex_step(xs, p, ys, p, eps, dt, 1e-13, U0)
    ref = U0 / (1 + 2 * np.pi ** 2 * dt * eps)
    err = np.sqrt(T.legendre_l2_sq(xs, p, ys, p, U1 - ref) / T.legendre_l2_sq(xs, p, ys, p, ref))
    assert err <= 1e-9, err


def test_imex_energy_decays_discontinuous_data():
    """Burgers with zero Dirichlet data dissipates: d/dt ||u||^2 =
    -2 eps ||grad u||^2 (the convective term is skew).  Piecewise constant
    initial data on 9 x 9 elements of (-1,1)^2 (the Fig. 'discont' setting,
    P:L780: 'resolve the right-hand side exactly'), eps = 0.1 (Fig. burgers
    caption)."""
    xs = ys = np.linspace(-1, 1, 10)
    p, eps, dt = 6, 0.1, 1e-3
    vals = np.random.default_rng(3).standard_normal((9, 9))
    U = np.zeros(((p + 1) * 9, (p + 1) * 9))
    U[:9, :9] = vals
    e0 = T.legendre_l2_sq(xs, p, ys, p, U)
    prev = e0
    for _ in range(4):
        U = T.imex_step(xs, p, ys, p, eps, dt, 1e-10, U)
        e = T.legendre_l2_sq(xs, p, ys, p, U)
        assert e < prev
        prev = e
    assert prev < 0.99 * e0
