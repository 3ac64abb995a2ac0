"""Seeded synthetic workloads shared by the tests, smoke() and bench.py.

This module holds the five BASELINE.json configurations and the seeded input
generators for them.  It contains none of the method's arithmetic (no basis
matrices, no factorisations, no ADI): it only produces

  * the meshes (breakpoints) of each configuration, and
  * the right-hand side f as piecewise-Legendre coefficients F_leg, the form
    in which the paper takes its data ("f_p computed via a fast
    Legendre transform or otherwise", "f are given Legendre
    coefficients").

Both the CUDA path (paper_2402_11299_b200) and the CPU oracle (oracle/)
consume these arrays; neither imports the other.  The input recipe and its
readings are stated in DESIGN.md "Inputs".

F_leg layout: ((p_x+1) n_x) x ((p_y+1) n_y), float64, row-major,
degree-major / element-minor in both dimensions: entry
[m*n_x + e, l*n_y + f] is the coefficient of P_m(x) P_l(y) on the element
(e, f) (the ordering of the paper's piecewise-Legendre quasi-matrix P,
P:L173-L176).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration (configs[idx-1])."""

    idx: int
    name: str
    ax: float
    bx: float
    ay: float
    by: float
    nx: int
    px: int
    ny: int
    py: int
    omega: float
    bc: int  # 0 = zero Dirichlet, 1 = zero Neumann
    tol: float
    mesh: str  # "uniform" or "graded"
    rhs: str  # "decay2", "decay2+spike", "singular+decay1.5"
    grading: float = 0.85

    @property
    def Nx(self) -> int:
        return (self.nx - 1 if self.bc == 0 else self.nx + 1) + (self.px - 1) * self.nx

    @property
    def Ny(self) -> int:
        return (self.ny - 1 if self.bc == 0 else self.ny + 1) + (self.py - 1) * self.ny

    @property
    def dofs(self) -> int:
        return self.Nx * self.Ny

    def breakpoints(self):
        return (_mesh(self.ax, self.bx, self.nx, self.mesh, self.grading),
                _mesh(self.ay, self.by, self.ny, self.mesh, self.grading))


CONFIGS = {
    1: Config(1, "dirichlet_unit_n4_p8", 0.0, 1.0, 0.0, 1.0, 4, 8, 4, 8, 0.0, 0, 1e-12, "uniform", "decay2"),
    2: Config(2, "dirichlet_unit_n16_p32", 0.0, 1.0, 0.0, 1.0, 16, 32, 16, 32, 0.0, 0, 1e-12, "uniform", "decay2"),
    3: Config(3, "screened10_dirichlet_pm1_n64_p64_spike", -1.0, 1.0, -1.0, 1.0, 64, 64, 64, 64, 10.0, 0, 1e-10,
              "uniform", "decay2+spike"),
    4: Config(4, "dirichlet_rect_x256p32_y32p256", 0.0, 2.0, 0.0, 1.0, 256, 32, 32, 256, 0.0, 0, 1e-12, "uniform",
              "decay2"),
    5: Config(5, "neumann_screened1_graded085_n128_p128_singular", 0.0, 1.0, 0.0, 1.0, 128, 128, 128, 128, 1.0, 1,
              1e-10, "graded", "singular+decay1.5"),
}


def _mesh(a: float, b: float, n: int, kind: str, sigma: float) -> np.ndarray:
    if kind == "uniform":
        return a + (b - a) * (np.arange(n + 1, dtype=np.float64) / n)
    if kind == "graded":
        # classical geometric mesh toward the left end: a, sigma^{n-1}, ..., sigma, 1
        # (scaled to [a, b]); reading R8
        t = np.empty(n + 1, dtype=np.float64)
        t[0] = 0.0
        t[1:] = sigma ** np.arange(n - 1, -1, -1, dtype=np.float64)
        return a + (b - a) * t
    raise ValueError(kind)


def uniform_mesh(a: float, b: float, n: int) -> np.ndarray:
    return _mesh(a, b, n, "uniform", 0.0)


def graded_mesh(a: float, b: float, n: int, sigma: float) -> np.ndarray:
    return _mesh(a, b, n, "graded", sigma)


# ---------------------------------------------------------------------------
# right-hand sides as piecewise-Legendre coefficients
# ---------------------------------------------------------------------------
def decay_field(rows_p: int, rows_n: int, cols_p: int, cols_n: int, seed: int, power: float) -> np.ndarray:
    """N(0,1) * (1+k)^-power * (1+l)^-power, k/l the LOCAL Legendre degree
    (reading R9), drawn with numpy default_rng(seed).standard_normal in
    row-major order of the degree-major F_leg array."""
    rng = np.random.default_rng(seed)
    F = rng.standard_normal(((rows_p + 1) * rows_n, (cols_p + 1) * cols_n))
    rk = (1.0 + np.repeat(np.arange(rows_p + 1, dtype=np.float64), rows_n)) ** (-power)
    ck = (1.0 + np.repeat(np.arange(cols_p + 1, dtype=np.float64), cols_n)) ** (-power)
    F *= rk[:, None]
    F *= ck[None, :]
    return F


def _legendre_table(p: int, t: np.ndarray) -> np.ndarray:
    """P_0..P_p at points t (three-term recurrence); shape (p+1, len(t))."""
    P = np.empty((p + 1, t.size))
    P[0] = 1.0
    if p >= 1:
        P[1] = t
    for k in range(1, p):
        P[k + 1] = ((2 * k + 1) * t * P[k] - k * P[k - 1]) / (k + 1)
    return P


def _analysis_1d(xs: np.ndarray, p: int, nq: int):
    """Gauss-Legendre analysis operator per element: returns (pts, V) with
    pts (n, nq) physical nodes and V (p+1, nq) = (2k+1)/2 P_k(t_q) w_q so
    that c_k = V @ f(pts[e]) is the degree-k Legendre coefficient."""
    t, w = np.polynomial.legendre.leggauss(nq)
    P = _legendre_table(p, t)
    V = P * w[None, :] * ((2.0 * np.arange(p + 1) + 1.0) / 2.0)[:, None]
    a, b = xs[:-1], xs[1:]
    pts = (a[:, None] + b[:, None]) / 2.0 + (b - a)[:, None] / 2.0 * t[None, :]
    return pts, V


def project_separable(xs, px, ys, py, fx, fy, nq_extra: int = 64) -> np.ndarray:
    """Piecewise-Legendre coefficients of f(x,y) = fx(x) fy(y)."""
    nx, ny = xs.size - 1, ys.size - 1
    px_pts, Vx = _analysis_1d(xs, px, px + 1 + nq_extra)
    py_pts, Vy = _analysis_1d(ys, py, py + 1 + nq_extra)
    cx = (Vx @ fx(px_pts).T)  # (px+1, nx)
    cy = (Vy @ fy(py_pts).T)  # (py+1, ny)
    return np.outer(cx.reshape(-1), cy.reshape(-1))  # degree-major / element-minor


def project_function(xs, px, ys, py, f, nq_extra: int = 64) -> np.ndarray:
    """Piecewise-Legendre coefficients of a general f(x, y) by tensor
    Gauss-Legendre quadrature with p+1+nq_extra points per direction."""
    nx, ny = xs.size - 1, ys.size - 1
    qx, qy = px + 1 + nq_extra, py + 1 + nq_extra
    xpts, Vx = _analysis_1d(xs, px, qx)
    ypts, Vy = _analysis_1d(ys, py, qy)
    out = np.empty(((px + 1) * nx, (py + 1) * ny))
    yflat = ypts.reshape(-1)
    for e in range(nx):
        vals = f(xpts[e][:, None], yflat[None, :])  # (qx, ny*qy)
        c1 = Vx @ vals  # (px+1, ny*qy)
        c2 = c1.reshape(px + 1, ny, qy) @ Vy.T  # (px+1, ny, py+1)
        out[e::nx, :] = c2.transpose(0, 2, 1).reshape(px + 1, (py + 1) * ny)
    return out


def f_leg(cfg: Config, seed: int = 0) -> np.ndarray:
    """The configuration's right-hand side as piecewise-Legendre coefficients
    (recipe: DESIGN.md "Inputs", readings R9-R11)."""
    xs, ys = cfg.breakpoints()
    if cfg.rhs == "decay2":
        return decay_field(cfg.px, cfg.nx, cfg.py, cfg.ny, seed, 2.0)
    if cfg.rhs == "decay2+spike":
        F = decay_field(cfg.px, cfg.nx, cfg.py, cfg.ny, seed, 2.0)
        s = 0.01
        g = 1.0 / (2.0 * math.pi * s * s)
        F += project_separable(xs, cfg.px, ys, cfg.py,
                               lambda x: g * np.exp(-(x - 0.3) ** 2 / (2 * s * s)),
                               lambda y: np.exp(-(y + 0.2) ** 2 / (2 * s * s)))
        return F
    if cfg.rhs == "singular+decay1.5":
        F = project_function(xs, cfg.px, ys, cfg.py, lambda x, y: (x * x + y * y) ** (-0.25))
        F += decay_field(cfg.px, cfg.nx, cfg.py, cfg.ny, seed, 1.5)
        return F
    raise ValueError(cfg.rhs)


def random_field(shape, seed: int) -> np.ndarray:
    """Plain seeded N(0,1) array (used for G / U test inputs)."""
    return np.random.default_rng(seed).standard_normal(shape)
