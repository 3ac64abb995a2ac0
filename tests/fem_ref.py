"""Independent reference FEM built from the paper's *definitions* by Gauss
quadrature -- used only to pin the oracle.

The basis is evaluated pointwise from P:L74
    W_k(x) = (1 - x^2) P_k^{(1,1)}(x) / (2 (k+1))
(scipy's Jacobi polynomials, not the App. A recurrence the oracle uses),
hats from P:L153-L166, the affine element maps from P:L143, the degree-major
ordering from P:L169-L171 and the Dirichlet restriction of P:L315.  Nothing
here calls the oracle or the CUDA path.
"""
from __future__ import annotations

import numpy as np
from scipy.special import eval_jacobi


def _ends(bc):
    """(left end Dirichlet?, right end Dirichlet?) for the 1D codes
    0 = Dirichlet, 1 = Neumann, 2 = Dirichlet/Neumann, 3 = Neumann/Dirichlet."""
    return {0: (True, True), 1: (False, False), 2: (True, False), 3: (False, True)}[bc]


def nhats(n, bc):
    dl, dr = _ends(bc)
    return n + 1 - int(dl) - int(dr)


def ndofs(n, p, bc):
    return nhats(n, bc) + (p - 1) * n


def hat_index(node, n, bc):
    dl, dr = _ends(bc)
    if (node == 0 and dl) or (node == n and dr):
        return -1
    return node - int(dl)


def bubble_ref(k, t):
    """W_k(t) on [-1,1] and its t-derivative (DLMF 18.9.15)."""
    Pk = eval_jacobi(k, 1, 1, t)
    dPk = 0.0 if k == 0 else (k + 3) / 2.0 * eval_jacobi(k - 1, 2, 2, t)
    W = (1 - t * t) * Pk / (2 * (k + 1))
    dW = (-2 * t * Pk + (1 - t * t) * dPk) / (2 * (k + 1))
    return W, dW


def basis_at(xs, p, bc, x):
    """Values and x-derivatives of all global basis functions at points x:
    returns (Phi, dPhi) of shape (len(x), N)."""
    xs = np.asarray(xs, dtype=np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = xs.size - 1
    N = ndofs(n, p, bc)
    nh = nhats(n, bc)
    Phi = np.zeros((x.size, N))
    dPhi = np.zeros((x.size, N))
    e_of = np.clip(np.searchsorted(xs, x, side="right") - 1, 0, n - 1)
    for e in range(n):
        sel = np.nonzero(e_of == e)[0]
        if sel.size == 0:
            continue
        a, b = xs[e], xs[e + 1]
        d = b - a
        t = (2 * x[sel] - a - b) / d  # affine map
        hl, hr = hat_index(e, n, bc), hat_index(e + 1, n, bc)
        if hl >= 0:
            Phi[sel, hl] += (b - x[sel]) / d
            dPhi[sel, hl] += -1.0 / d
        if hr >= 0:
            Phi[sel, hr] += (x[sel] - a) / d
            dPhi[sel, hr] += 1.0 / d
        for k in range(p - 1):
            W, dW = bubble_ref(k, t)
            Phi[sel, nh + k * n + e] = W
            dPhi[sel, nh + k * n + e] = dW * 2.0 / d
    return Phi, dPhi


def quad_points(xs, nq):
    """Composite Gauss-Legendre nodes / weights on the mesh."""
    t, w = np.polynomial.legendre.leggauss(nq)
    xs = np.asarray(xs, dtype=np.float64)
    a, b = xs[:-1], xs[1:]
    pts = ((a + b)[:, None] + (b - a)[:, None] * t[None, :]) / 2
    wts = (b - a)[:, None] / 2 * w[None, :]
    return pts.reshape(-1), wts.reshape(-1)


def assemble_quad(xs, p, bc):
    """(K, M) = (<phi_i', phi_j'>, <phi_i, phi_j>) by quadrature (exact for
    these polynomial degrees)."""
    x, w = quad_points(xs, p + 3)
    Phi, dPhi = basis_at(xs, p, bc, x)
    M = Phi.T @ (w[:, None] * Phi)
    K = dPhi.T @ (w[:, None] * dPhi)
    return K, M


def legendre_eval(xs, p, c, x):
    """Evaluate a piecewise-Legendre expansion (coefficient index m*n + e)."""
    xs = np.asarray(xs, dtype=np.float64)
    n = xs.size - 1
    e_of = np.clip(np.searchsorted(xs, x, side="right") - 1, 0, n - 1)
    a, b = xs[e_of], xs[e_of + 1]
    t = (2 * x - a - b) / (b - a)
    out = np.zeros((x.size,) + np.shape(c)[1:])
    for m in range(p + 1):
        Pm = eval_jacobi(m, 0, 0, t)
        out += (Pm * 1.0)[:, None] * c[m * n + e_of] if np.ndim(c) > 1 else Pm * c[m * n + e_of]
    return out


def legendre_basis_at(xs, p, x):
    """Matrix of piecewise Legendre functions P_{m,e}(x): (len(x), (p+1) n)."""
    xs = np.asarray(xs, dtype=np.float64)
    n = xs.size - 1
    e_of = np.clip(np.searchsorted(xs, x, side="right") - 1, 0, n - 1)
    a, b = xs[e_of], xs[e_of + 1]
    t = (2 * x - a - b) / (b - a)
    B = np.zeros((x.size, (p + 1) * n))
    for m in range(p + 1):
        B[np.arange(x.size), m * n + e_of] = eval_jacobi(m, 0, 0, t)
    return B
