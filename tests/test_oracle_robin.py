"""Pins of the oracle's Robin ends (alpha u + du/dn = 0 on a
side, discretised in the full basis C with the boundary term
alpha <v, u>_{L2(side)}; NEXT-1 of SURVEY 8(f)).  CPU only."""
import numpy as np
import pytest
import scipy.linalg as sla
from scipy.optimize import brentq

import fem_ref
import oracle


def rand_mesh(n, a=0.0, b=1.0, seed=0):
    w = np.random.default_rng(seed).uniform(0.3, 1.7, size=n)
    xs = np.concatenate([[0.0], np.cumsum(w)])
    return a + (b - a) * xs / xs[-1]


@pytest.mark.parametrize("bc,al,ar", [(1, 2.0, 0.5), (1, 0.0, 3.0), (2, 0.0, 1.5), (3, 4.0, 0.0)])
def test_robin_boundary_term(bc, al, ar):
    """K_Robin - K = alpha_a phi(a) phi(a)^T + alpha_b phi(b) phi(b)^T, the
    boundary integral of the variational form, with the basis
    evaluated at the ends by fem_ref (Jacobi-defined bubbles)."""
    xs = rand_mesh(4, 0.0, 2.0, seed=1)
    p = 5
    K0 = oracle.operator_dense(xs, p, bc, 1.0, 0.0)
    with oracle.robin([al, ar, 0.0, 0.0]):
        K1 = oracle.operator_dense(xs, p, bc, 1.0, 0.0)
        M1 = oracle.operator_dense(xs, p, bc, 0.0, 1.0)
    pa = fem_ref.basis_at(xs, p, bc, np.array([xs[0]]))[0][0]
    pb = fem_ref.basis_at(xs, p, bc, np.array([xs[-1]]))[0][0]
    np.testing.assert_allclose(K1 - K0, al * np.outer(pa, pa) + ar * np.outer(pb, pb), atol=1e-13)
    np.testing.assert_array_equal(M1, oracle.operator_dense(xs, p, bc, 0.0, 1.0))


def robin_eig1(L, al, ar):
    """First eigenvalue k^2 of -u'' = k^2 u on [0, L] with al u - u' = 0 at 0
    and ar u + u' = 0 at L: u = cos kx + (al/k) sin kx,
    (al ar - k^2) sin kL + k (al + ar) cos kL = 0, first root."""
    f = lambda k: (al * ar - k * k) * np.sin(k * L) + k * (al + ar) * np.cos(k * L)
    ks = np.linspace(1e-9, np.pi / L, 2000)
    v = f(ks)
    i = np.nonzero(np.sign(v[:-1]) != np.sign(v[1:]))[0][0]
    k = brentq(f, ks[i], ks[i + 1], xtol=1e-15)
    return k * k


@pytest.mark.parametrize("al,ar,om", [(3.0, 3.0, 0.0), (0.5, 2.0, 0.0), (1.0, 0.0, 0.0), (2.0, 1.0, 1.5)])
def test_robin_lambda_min(al, ar, om):
    """The oracle's lambda_min (bisection, reading R22) matches the dense
    generalised eigenvalue (scipy eigh) and, at p = 12, the continuous first
    eigenvalue of the Robin problem (+ w^2/2) to spectral accuracy, from
    above (conforming Galerkin)."""
    xs = rand_mesh(3, 0.0, 1.0, seed=2)
    p = 12
    with oracle.robin([al, ar, 0.0, 0.0]):
        lam = oracle.spectrum(xs, p, 1, om)
        K = oracle.operator_dense(xs, p, 1, 1.0, 0.0)
        M = oracle.operator_dense(xs, p, 1, 0.0, 1.0)
    ev = sla.eigh(K + om * om / 2 * M, M, eigvals_only=True)
    # the SPD test near lambda_min resolves it to ~ eps lambda_max / lambda_min
    # relative (1.3e-11 measured here; eigh carries the same ~ eps lambda_max)
    assert abs(lam[0] - ev[0]) <= 1e-10 * ev[0]
    assert abs(lam[1] - ev[-1]) <= 1e-11 * ev[-1] and lam[1] >= ev[-1]
    lc = robin_eig1(1.0, al, ar) + om * om / 2
    assert lc <= ev[0] * (1 + 1e-10) and ev[0] - lc <= 1e-9 * lc  # from above, to the eigh rounding level


def test_robin_alpha_zero_is_neumann():
    xs = rand_mesh(3, seed=3)
    G = np.random.default_rng(4).standard_normal((oracle.dim(3, 5, 1), oracle.dim(3, 5, 1)))
    U0, J0 = oracle.adi_solve(xs, 5, xs, 5, 1.0, 1, 1e-10, G)
    with oracle.robin([0.0, 0.0, 0.0, 0.0]):
        U1, J1 = oracle.adi_solve(xs, 5, xs, 5, 1.0, 1, 1e-10, G)
    assert J0 == J1 and np.array_equal(U0, U1)


def test_robin_rejects_dirichlet_end_and_negative_alpha():
    xs = rand_mesh(2, seed=5)
    with oracle.robin([1.0, 0.0, 0.0, 0.0]):
        with pytest.raises(oracle.OracleError):
            oracle.operator_dense(xs, 4, 0, 1.0, 0.0)  # Dirichlet left end
    with oracle.robin([-1.0, 0.0, 0.0, 0.0]):
        with pytest.raises(oracle.OracleError):
            oracle.operator_dense(xs, 4, 1, 1.0, 0.0)


def robin_mode(k):
    """(alpha, v): v(x) = cos kx + (alpha/k) sin kx on [0,1] satisfies
    alpha v - v' = 0 at 0 and alpha v + v' = 0 at 1 for
    alpha = k (1 - cos k)/sin k, and -v'' = k^2 v."""
    al = k * (1 - np.cos(k)) / np.sin(k)
    return al, (lambda x: np.cos(k * x) + al / k * np.sin(k * x))


@pytest.mark.parametrize("om", [0.0, 2.0])
def test_robin_manufactured_2d(om):
    """u = v(x) v(y) with the Robin mode v: -Delta u + w^2 u = (2k^2 + w^2) u
    with Robin conditions on all four sides.  Load the projected f, ADI
    solve, and compare the L2 error against the exact u: exponential
    convergence in p (p = 4 -> 12)."""
    k = 2.0
    al, v = robin_mode(k)
    lam = 2 * k * k + om * om
    xs = rand_mesh(2, seed=6)
    errs = []
    for p in (4, 8, 12):
        tq, wq = np.polynomial.legendre.leggauss(p + 30)
        cv = np.zeros((p + 1) * 2)
        for e in range(2):
            x = xs[e] + (tq + 1) * (xs[e + 1] - xs[e]) / 2
            for m in range(p + 1):
                Pm = np.polynomial.legendre.legval(tq, np.eye(m + 1)[m])
                cv[m * 2 + e] = (2 * m + 1) / 2 * np.sum(wq * Pm * v(x))
        Cu = np.outer(cv, cv)
        with oracle.robin([al, al, al, al]):
            G = oracle.load(xs, p, xs, p, 1, lam * Cu)
            U, _ = oracle.adi_solve(xs, p, xs, p, om, 1, 1e-13, G)
        C = oracle.unload(xs, p, xs, p, 1, U)
        wts = np.array([(xs[e + 1] - xs[e]) / (2 * m + 1) for m in range(p + 1) for e in range(2)])
        errs.append(float(np.sqrt(np.einsum("i,j,ij->", wts, wts, (C - Cu) ** 2))))
    assert errs[1] < 1e-3 * errs[0] and errs[2] < 1e-9, errs
