"""Pins of the CPU oracle against what the paper and mathematics fix
(never against the oracle's own formulas, never against the CUDA path).

Each test names the passage (P:Lnnn = PAPER.md line, S:Lnnn = SPEC.md line)
or the mathematical fact it checks.  CPU only (-m "not gpu").
"""
import math

import mpmath as mp
import numpy as np
import pytest
import scipy.linalg as sla

import fem_ref
import oracle
import workloads as W

RNG = np.random.default_rng(1234)


def rand_mesh(n, a=0.0, b=1.0, rng=RNG):
    w = rng.uniform(0.3, 1.7, size=n)
    xs = np.concatenate([[0.0], np.cumsum(w)])
    return a + (b - a) * xs / xs[-1]


MESHES = [
    (np.array([-1.0, 1.0]), 5),
    (np.linspace(0, 1, 4), 4),
    (rand_mesh(5), 6),
    (rand_mesh(3, -1, 2), 2),
    (W.graded_mesh(0, 1, 6, 0.5), 7),
]


# ---------------------------------------------------------------- operators
def test_reference_element_values():
    """Single element [-1,1]: -Delta_W = diag(2/(2k+3)) and
    <W_0,W_0> = 2/9 + 2/45 (from the lowering L_W^T M_P L_W P:L120)."""
    xs = np.array([-1.0, 1.0])
    K = oracle.operator_dense(xs, 6, 0, 1.0, 0.0)  # Dirichlet n=1: bubbles only
    M = oracle.operator_dense(xs, 6, 0, 0.0, 1.0)
    np.testing.assert_allclose(np.diag(K), [2 / (2 * k + 3) for k in range(5)], rtol=1e-15)
    assert np.count_nonzero(K - np.diag(np.diag(K))) == 0
    assert M[0, 0] == pytest.approx(2 / 9 + 2 / 45, rel=1e-15)
    # odd offsets vanish exactly (parity)
    for i in range(5):
        for j in range(5):
            if (i - j) % 2 == 1:
                assert M[i, j] == 0.0


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
@pytest.mark.parametrize("mi", range(len(MESHES)))
def test_operators_vs_quadrature(mi, bc):
    """K = <phi', phi'>, M = <phi, phi> against Gauss
    quadrature with the Jacobi definition of W_k."""
    xs, p = MESHES[mi]
    if bc != 1 and xs.size == 2 and p < 2:
        pytest.skip()
    Kq, Mq = fem_ref.assemble_quad(xs, p, bc)
    K = oracle.operator_dense(xs, p, bc, 1.0, 0.0)
    M = oracle.operator_dense(xs, p, bc, 0.0, 1.0)
    assert np.abs(M - Mq).max() <= 1e-14 * np.abs(Mq).max()
    assert np.abs(K - Kq).max() <= 1e-12 * np.abs(Kq).max()


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_b3_sparsity(bc):
    """B^3-Arrowhead structure (Def. 4.1): K tridiagonal on hats
    and diagonal on bubbles; in M every block outside the first
    block row/column is diagonal, and hats only couple to bubble
    degrees 0 and 1."""
    xs, p = rand_mesh(5), 7
    n = xs.size - 1
    nh = fem_ref.nhats(n, bc)
    K = oracle.operator_dense(xs, p, bc, 1.0, 0.0)
    M = oracle.operator_dense(xs, p, bc, 0.0, 1.0)
    N = K.shape[0]
    for i in range(N):
        for j in range(N):
            ih, jh = i < nh, j < nh
            if ih and jh:
                if abs(i - j) > 1:
                    assert K[i, j] == 0 and M[i, j] == 0
            elif ih != jh:
                assert K[i, j] == 0
                b = j if ih else i
                k = (b - nh) // n
                if k >= 2:
                    assert M[i, j] == 0
            else:
                if i != j:
                    assert K[i, j] == 0
                ki, ei = divmod(i - nh, n)
                kj, ej = divmod(j - nh, n)
                if ei != ej or abs(ki - kj) not in (0, 2):
                    assert M[i, j] == 0


def test_dimension_formula():
    """N = p n - 1 (Dirichlet); p n + 1 for the full basis C; p n
    with one Dirichlet and one Neumann end (mixed, NEXT-1)."""
    for n, p in [(1, 2), (4, 8), (16, 32), (3, 5)]:
        assert oracle.dim(n, p, 0) == p * n - 1
        assert oracle.dim(n, p, 1) == p * n + 1
        assert oracle.dim(n, p, 2) == p * n
        assert oracle.dim(n, p, 3) == p * n


# --------------------------------------------------------- reverse Cholesky
FACTOR_CASES = [
    (rand_mesh(4), 6, 0, 1.0, 3.7),
    (rand_mesh(5), 5, 1, 1.0, 0.9),
    (np.array([0.0, 1.0]), 7, 0, 1.0, 0.0),
    (np.array([0.0, 1.0]), 2, 1, 1.0, 2.0),
    (W.graded_mesh(0, 1, 7, 0.4), 8, 1, 1.0, 0.5),
    (rand_mesh(3), 4, 0, 0.0, 1.0),  # mass only
]


@pytest.mark.parametrize("case", range(len(FACTOR_CASES)))
def test_reverse_cholesky(case):
    """Thm 4.2 / Alg. 1: A = L^T L, L lower triangular with the
    sparsity of tril(A) (zero fill), and L equals the dense reverse
    Cholesky flip(chol(flip A flip)) flip."""
    xs, p, bc, al, be = FACTOR_CASES[case]
    A = oracle.operator_dense(xs, p, bc, al, be)
    L = oracle.factor_dense(xs, p, bc, al, be)
    assert np.allclose(L, np.tril(L), atol=0)
    assert np.linalg.norm(L.T @ L - A) <= 1e-14 * np.linalg.norm(A) * max(1, A.shape[0] ** 0.5)
    assert not np.any((L != 0) & (np.tril(A) == 0)), "fill-in outside tril(A)"
    F = np.flipud(np.fliplr(A))
    Ld = np.flipud(np.fliplr(np.linalg.cholesky(F)))
    Ld = Ld.T  # flip(chol) is upper -> L^T L form
    assert np.abs(L - Ld).max() <= 1e-12 * np.abs(Ld).max()


def test_not_positive_definite():
    """A non-positive pivot is reported, not hidden."""
    xs = rand_mesh(3)
    with pytest.raises(oracle.OracleError):
        oracle.factor_dense(xs, 5, 0, -1.0, 0.0)  # -K is negative definite


@pytest.mark.parametrize("case", range(len(FACTOR_CASES)))
def test_solve1d_vs_lapack(case):
    """Cor. 4.3 O(N) solve equals the dense LAPACK solve."""
    xs, p, bc, al, be = FACTOR_CASES[case]
    A = oracle.operator_dense(xs, p, bc, al, be)
    f = RNG.standard_normal((3, A.shape[0]))
    x = oracle.solve1d(xs, p, bc, al, be, f)
    xd = np.linalg.solve(A, f.T).T
    cond = np.linalg.cond(A)
    assert np.abs(x - xd).max() <= 1e-15 * cond * np.abs(xd).max() * 10


# ------------------------------------------------------- spectral interval
SPEC_CASES = [
    (np.linspace(0, 1, 5), 8, 0, 0.0),
    (np.linspace(-1, 1, 4), 6, 0, 10.0),
    (rand_mesh(4, 0, 2), 5, 1, 1.0),
    (W.graded_mesh(0, 1, 8, 0.5), 6, 1, 1.0),
    (np.linspace(0, 1, 3), 3, 1, 3.0),
    (rand_mesh(5, 0, 2), 6, 2, 0.0),  # mixed Dirichlet / Neumann
    (W.graded_mesh(0, 1, 6, 0.5), 5, 3, 2.0),
]


@pytest.mark.parametrize("case", range(len(SPEC_CASES)))
def test_spectrum_vs_eigh(case):
    """Extreme generalised eigenvalues of (A, M), A = K + w^2/2 M
    (Alg. 2 line 1): the oracle's interval contains the dense
    LAPACK spectrum and is tight (reading R4)."""
    xs, p, bc, om = SPEC_CASES[case]
    K = oracle.operator_dense(xs, p, bc, 1.0, 0.0)
    M = oracle.operator_dense(xs, p, bc, 0.0, 1.0)
    ev = sla.eigh(K + om * om / 2 * M, M, eigvals_only=True)
    lam = oracle.spectrum(xs, p, bc, om)
    # dense LAPACK is itself only accurate to ~u*cond(M) on graded meshes
    slack = 1e-12 if bc == 0 else 1e-13 * np.linalg.cond(M)
    assert lam[0] <= ev[0] * (1 + slack)
    assert lam[1] >= ev[-1] * (1 - 1e-12)
    assert lam[1] <= ev[-1] * (1 + 1e-9)
    if bc == 1:
        # the constant function (all hats 1, bubbles 0) is an exact eigenvector
        # with eigenvalue w^2/2 since K c = 0 (constants are in C)
        n = xs.size - 1
        c = np.zeros(K.shape[0])
        c[: n + 1] = 1.0
        assert np.abs(K @ c).max() <= 1e-13 * np.abs(K).max()
        assert lam[0] == pytest.approx(om * om / 2, rel=1e-15)
    elif bc == 0:
        # Poincare: discrete lambda_min >= pi^2/L^2 + w^2/2
        L = xs[-1] - xs[0]
        assert lam[0] == pytest.approx(math.pi ** 2 / L ** 2 + om * om / 2, rel=1e-15)
    else:
        # mixed ends: the continuous first eigenvalue is the quarter wave
        # pi^2/(4 L^2) + w^2/2, a lower bound of the conforming discrete one
        L = xs[-1] - xs[0]
        assert lam[0] == pytest.approx(math.pi ** 2 / (4 * L ** 2) + om * om / 2, rel=1e-15)
        assert ev[0] <= lam[0] * (1 + 1e-2)  # and close to it at this resolution


@pytest.mark.parametrize("case", range(len(SPEC_CASES)))
def test_lemma52_containment(case):
    """Lemma 5.2: sigma(L^-T M L^-1) in [2h^2/(24p^4 + w^2 h^2), C]."""
    xs, p, bc, om = SPEC_CASES[case]
    h = np.diff(xs).min()
    L = xs[-1] - xs[0]
    lam = oracle.spectrum(xs, p, bc, om)  # of (A, M): sigma(L^-T M L^-1) = 1/lam
    lo = 2 * h * h / (24 * p ** 4 + om * om * h * h)
    if bc == 0:
        C = min(L * L / math.pi ** 2, max(1.0, 2.0 / om ** 2) if om else math.inf)
    elif bc == 1:
        C = max(1.0, 2.0 / om ** 2)
    else:  # mixed ends: the quarter-wave Poincare constant (4 L^2 / pi^2)
        C = min(4 * L * L / math.pi ** 2, max(1.0, 2.0 / om ** 2) if om else math.inf)
    assert 1.0 / lam[1] >= lo * (1 - 1e-12)
    assert 1.0 / lam[0] <= C * (1 + 1e-12)


# ----------------------------------------------------------- J and shifts
def test_J_formula_example():
    """J = ceil(log(16 gamma) log(4/eps)/pi^2); gamma = 10,
    eps = 1e-4 gives J = 6."""
    b = 19 + math.sqrt(360)  # symmetric [1,b], [-b,-1]: gamma = (1+b)^2/(4b) = 10
    J, g, P, Q = oracle.shifts(1.0, b, -b, -1.0, 1e-4)
    assert g == pytest.approx(10.0, rel=1e-14)
    assert J == 6


def _mp_shifts(a, b, c, d, J, dps=140):
    mp.mp.dps = dps
    a, b, c, d = map(mp.mpf, (a, b, c, d))
    g = abs(c - a) * abs(d - b) / (abs(c - b) * abs(d - a))
    al = -1 + 2 * g + 2 * mp.sqrt(g * g - g)
    m = 1 - 1 / al ** 2
    K = mp.ellipk(m) if m > 0 else mp.pi / 2

    def T(z):  # Moebius with T(-al)=a, T(-1)=b, T(1)=c (cross ratio)
        rho = (z + al) * (-2) / ((z - 1) * (al - 1))
        return (a * (b - c) - rho * c * (b - a)) / ((b - c) - rho * (b - a))

    P, Q = [], []
    for j in range(1, J + 1):
        u = (2 * j - 1) * K / (2 * J)
        dn = mp.ellipfun("dn", u, m=m) if m > 0 else mp.mpf(1)
        P.append(T(-al * dn))
        Q.append(T(al * dn))
    return P, Q


SHIFT_CASES = [
    (math.pi ** 2, 50310.4545546266, 1e-12),  # config 1 interval
    (0.5, 2.6108637024878e27, 1e-10),  # config 5 interval (k' ~ 2e-28)
    (1.0, 1e16, 1e-8),  # k' ~ 2.5e-17: the sech branch
    (1.0, 2.5e7, 1e-6),  # k' ~ 1e-8: branch boundary
    (1.0, 3.0, 1e-12),  # moderate modulus
]


@pytest.mark.parametrize("case", range(len(SHIFT_CASES)))
def test_shifts_symmetric_vs_mpmath(case):
    """Zolotarev shifts (reading R5) against mpmath's elliptic dn at
    140 digits; p_j > 0, q_j < 0."""
    a, b, eps = SHIFT_CASES[case]
    J, g, P, Q = oracle.shifts(a, b, -b, -a, eps)
    Pm, Qm = _mp_shifts(a, b, -b, -a, J)
    assert np.all(P > 0) and np.all(Q < 0)
    for j in range(J):
        assert abs(P[j] - float(Pm[j])) <= 4e-16 * abs(float(Pm[j]))
        assert abs(Q[j] - float(Qm[j])) <= 4e-16 * abs(float(Qm[j]))
    # reflection dn(K-u) dn(u) = k'  =>  p_j p_{J+1-j} = a b
    for j in range(J):
        assert P[j] * P[J - 1 - j] == pytest.approx(a * b, rel=1e-14)


def test_shifts_asymmetric_vs_mpmath():
    """General Moebius case (config 4 intervals)."""
    a, b = 2.4674011002723395, 8371393546.959874
    c, d = -1824569548969.281, -9.869604401089358
    J, g, P, Q = oracle.shifts(a, b, c, d, 1e-12)
    assert J == 68
    Pm, Qm = _mp_shifts(a, b, c, d, J)
    assert np.all((P >= a) & (P <= b)) and np.all((Q >= c) & (Q <= d))
    for j in range(J):
        assert abs(P[j] - float(Pm[j])) <= 1e-14 * abs(float(Pm[j]))
        assert abs(Q[j] - float(Qm[j])) <= 1e-14 * abs(float(Qm[j]))


def test_config_plans_J():
    """J per configuration (exact-eigenvalue column):
    30, 53, 50, 68, 162."""
    for i, J in [(1, 30), (2, 53), (3, 50), (4, 68), (5, 162)]:
        c = W.CONFIGS[i]
        xs, ys = c.breakpoints()
        pl = oracle.plan(xs, c.px, ys, c.py, c.omega, c.bc, c.tol)
        assert pl["J"] == J, (i, pl["J"])
        assert pl["Nx"] == c.Nx and pl["Ny"] == c.Ny


def test_neumann_J_nonincreasing_in_omega():
    """Fig. 5: cost falls as omega grows."""
    xs = np.linspace(0, 1, 3)
    Js = [oracle.plan(xs, 16, xs, 16, om, 1, 1e-10)["J"] for om in (0.5, 1.0, 10.0, 100.0)]
    assert all(Js[i + 1] <= Js[i] for i in range(len(Js) - 1)), Js


# --------------------------------------------------------------------- ADI
ADI_CASES = [
    (np.linspace(0, 1, 4), 5, np.linspace(0, 1, 4), 5, 0.0, 0),
    (np.linspace(0, 1, 3), 6, np.linspace(0, 2, 4), 4, 3.0, 0),
    (rand_mesh(3), 5, rand_mesh(2, 0, 3), 6, 1.0, 1),
    (W.graded_mesh(0, 1, 6, 0.5), 5, W.graded_mesh(0, 1, 6, 0.5), 5, 1.0, 1),
    (np.linspace(-1, 1, 3), 7, np.linspace(-1, 1, 3), 7, 10.0, 0),
    (rand_mesh(3), 6, rand_mesh(4, 0, 2), 5, 0.0, oracle.bc2d(2, 3)),  # mixed ends, per direction (NEXT-1)
]


def _dense_sylvester(xs, px, ys, py, om, bc, G):
    bx, by = oracle.split_bc(bc)
    Kx, Mx = oracle.operator_dense(xs, px, bx, 1, 0), oracle.operator_dense(xs, px, bx, 0, 1)
    Ky, My = oracle.operator_dense(ys, py, by, 1, 0), oracle.operator_dense(ys, py, by, 0, 1)
    Ax, Ay = Kx + om * om / 2 * Mx, Ky + om * om / 2 * My
    Big = np.kron(Ax, My) + np.kron(Mx, Ay)  # vec_row(A_x U M_y + M_x U A_y)
    U = np.linalg.solve(Big, G.reshape(-1)).reshape(G.shape)
    return U, Mx, My, Ax, Ay


@pytest.mark.parametrize("tol", [1e-2, 1e-4, 1e-8, 1e-12])
@pytest.mark.parametrize("case", range(len(ADI_CASES)))
def test_adi_lemma51(case, tol):
    """Lemma 5.1: ||V(U - U_J)L^T|| <= eps ||V U L^T||,
    M_x = V^T V, M_y = L^T L, U the dense Kronecker solution of
    eq. adi:poisson."""
    xs, px, ys, py, om, bc = ADI_CASES[case]
    Nx, Ny = oracle.dim(xs.size - 1, px, oracle.split_bc(bc)[0]), oracle.dim(ys.size - 1, py, oracle.split_bc(bc)[1])
    G = RNG.standard_normal((Nx, Ny))
    Us, Mx, My, _, _ = _dense_sylvester(xs, px, ys, py, om, bc, G)
    U, J = oracle.adi_solve(xs, px, ys, py, om, bc, tol, G)
    V = np.linalg.cholesky(Mx).T
    L = np.linalg.cholesky(My).T
    err = np.linalg.norm(V @ (U - Us) @ L.T, 2)
    ref = np.linalg.norm(V @ Us @ L.T, 2)
    floor = 1e-13 * np.linalg.cond(Mx) * np.linalg.cond(My)  # fp64 floor on these tiny cases
    assert err <= tol * ref + floor * ref, (err / ref, tol)


def test_adi_contraction_per_J():
    """The bound the J formula inverts: after J' iterations (shifts built
    for J'), err <= 4 exp(-pi^2 J'/log(16 gamma)) (FT20 Th. 2.1 as used at
    P:L751-L753)."""
    xs, px, ys, py, om, bc = ADI_CASES[0]
    Nx, Ny = oracle.dim(xs.size - 1, px, oracle.split_bc(bc)[0]), oracle.dim(ys.size - 1, py, oracle.split_bc(bc)[1])
    G = RNG.standard_normal((Nx, Ny))
    Us, Mx, My, _, _ = _dense_sylvester(xs, px, ys, py, om, bc, G)
    V, L = np.linalg.cholesky(Mx).T, np.linalg.cholesky(My).T
    g = oracle.plan(xs, px, ys, py, om, bc, 0.5)["gamma"]
    seen = set()
    for k in range(1, 40):
        eps = 4 * math.exp(-math.pi ** 2 * k / math.log(16 * g))  # J(eps) == k up to rounding
        U, J = oracle.adi_solve(xs, px, ys, py, om, bc, min(eps * 1.0000001, 0.99), G)
        if J in seen:
            continue
        seen.add(J)
        bound = 4 * math.exp(-math.pi ** 2 * J / math.log(16 * g))
        err = np.linalg.norm(V @ (U - Us) @ L.T, 2) / np.linalg.norm(V @ Us @ L.T, 2)
        assert err <= max(bound, 1e-12) * (1 + 1e-9), (J, err, bound)
    assert len(seen) >= 10


@pytest.mark.parametrize("swap", [False, True])
def test_adi_one_point_spectrum(swap):
    """Reading R15: N = 1 in exactly one direction (a one-point interval, the
    Moebius map of R5 degenerates).  The shift at that point makes the ADI
    error factor (z - p)/(z - q) vanish there, so the FIRST iteration is
    already the dense Kronecker solution to rounding; the
    shifts are finite with p > 0 > q."""
    a = (rand_mesh(1), 2)           # N = 1 (Dirichlet, one element, p = 2)
    b = (rand_mesh(3, 0, 2), 4)     # N = 11
    (xs, px), (ys, py) = (b, a) if swap else (a, b)
    om, bc = 0.7, 0
    Nx, Ny = oracle.dim(xs.size - 1, px, oracle.split_bc(bc)[0]), oracle.dim(ys.size - 1, py, oracle.split_bc(bc)[1])
    G = RNG.standard_normal((Nx, Ny))
    Us, _, _, _, _ = _dense_sylvester(xs, px, ys, py, om, bc, G)
    pl = oracle.plan(xs, px, ys, py, om, bc, 1e-10)
    assert np.all(np.isfinite(pl["p"])) and np.all(pl["p"] > 0) and np.all(pl["q"] < 0)
    U1, _ = oracle.adi_solve(xs, px, ys, py, om, bc, 1e-10, G, iters=1)
    assert np.abs(U1 - Us).max() <= 1e-12 * np.abs(Us).max()


def test_adi_1x1():
    """n = 1, p = 2, Dirichlet: N = 1 (no hats), gamma = 1 and the
    first iteration is exact: U = G / (2 a m) with, on the reference
    element, m = 2/9 + 2/45 and a = 2/3 + w^2/2 m."""
    xs = np.array([-1.0, 1.0])
    for om in (0.0, 2.0):
        G = np.array([[1.7]])
        U, J = oracle.adi_solve(xs, 2, xs, 2, om, 0, 1e-10, G)
        m = 2 / 9 + 2 / 45
        a = 2 / 3 + om * om / 2 * m
        assert U[0, 0] == pytest.approx(1.7 / (2 * a * m), rel=1e-14)


def test_adi_zero_and_linear():
    """F = 0 => U = 0; the solve is linear in F."""
    xs, px, ys, py, om, bc = ADI_CASES[2]
    Nx, Ny = oracle.dim(xs.size - 1, px, oracle.split_bc(bc)[0]), oracle.dim(ys.size - 1, py, oracle.split_bc(bc)[1])
    U0, _ = oracle.adi_solve(xs, px, ys, py, om, bc, 1e-10, np.zeros((Nx, Ny)))
    assert np.all(U0 == 0)
    G1, G2 = RNG.standard_normal((2, Nx, Ny))
    U1, _ = oracle.adi_solve(xs, px, ys, py, om, bc, 1e-10, G1)
    U2, _ = oracle.adi_solve(xs, px, ys, py, om, bc, 1e-10, G2)
    U3, _ = oracle.adi_solve(xs, px, ys, py, om, bc, 1e-10, 2 * G1 - 3 * G2)
    assert np.abs(U3 - (2 * U1 - 3 * U2)).max() <= 1e-12 * np.abs(U3).max()


# ------------------------------------------------------------ apply / load
@pytest.mark.parametrize("case", range(len(ADI_CASES)))
def test_apply_vs_dense(case):
    """A_x U M_y + M_x U A_y equals the dense Kronecker matvec built from
    the quadrature operators."""
    xs, px, ys, py, om, bc = ADI_CASES[case]
    bx, by = oracle.split_bc(bc)
    Kx, Mx = fem_ref.assemble_quad(xs, px, bx)
    Ky, My = fem_ref.assemble_quad(ys, py, by)
    Ax, Ay = Kx + om * om / 2 * Mx, Ky + om * om / 2 * My
    U = RNG.standard_normal((Kx.shape[0], Ky.shape[0]))
    F = oracle.apply(xs, px, ys, py, om, bc, U)
    Fd = Ax @ U @ My + Mx @ U @ Ay
    assert np.abs(F - Fd).max() <= 1e-12 * np.abs(Fd).max()


def test_load_constant_one():
    """f = 1 on one element [-1,1]: <W_0, 1> = 2/3; other bubbles
    integrate to 0; Neumann hats integrate to 1 each."""
    xs = np.array([-1.0, 1.0])
    p = 5
    Fleg = np.zeros(((p + 1), (p + 1)))
    Fleg[0, 0] = 1.0  # f(x,y) = 1
    G = oracle.load(xs, p, xs, p, 0, Fleg)
    g1 = np.zeros(p - 1)
    g1[0] = 2 / 3
    np.testing.assert_allclose(G, np.outer(g1, g1), atol=1e-16)
    G = oracle.load(xs, p, xs, p, 1, Fleg)
    g1 = np.concatenate([[1.0, 1.0], [2 / 3], np.zeros(p - 2)])
    np.testing.assert_allclose(G, np.outer(g1, g1), atol=1e-15)


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_load_vs_quadrature(bc):
    """G_ij = <phi_i psi_j, f> for a random
    piecewise-polynomial f, by tensor quadrature."""
    xs, px = rand_mesh(3), 5
    ys, py = rand_mesh(2, 0, 2), 4
    nx, ny = xs.size - 1, ys.size - 1
    Fleg = RNG.standard_normal(((px + 1) * nx, (py + 1) * ny))
    G = oracle.load(xs, px, ys, py, bc, Fleg)
    x, wx = fem_ref.quad_points(xs, px + 3)
    y, wy = fem_ref.quad_points(ys, py + 3)
    Px, _ = fem_ref.basis_at(xs, px, bc, x)
    Py, _ = fem_ref.basis_at(ys, py, bc, y)
    Lx = fem_ref.legendre_basis_at(xs, px, x)
    Ly = fem_ref.legendre_basis_at(ys, py, y)
    fvals = Lx @ Fleg @ Ly.T
    Gq = (Px * wx[:, None]).T @ fvals @ (Py * wy[:, None])
    assert np.abs(G - Gq).max() <= 1e-13 * np.abs(Gq).max()


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_unload_pointwise(bc):
    """C_leg = R_x U R_y^T reproduces the FEM function pointwise: the
    Legendre series with coefficients C_leg equals sum U_ij phi_i(x) psi_j(y)
    (basis evaluated from the Jacobi definition of W_k) at random
    points (NEXT-1 of SURVEY 8(f))."""
    xs, px = rand_mesh(3), 6
    ys, py = rand_mesh(2, 0, 2), 5
    Nx, Ny = fem_ref.ndofs(xs.size - 1, px, bc), fem_ref.ndofs(ys.size - 1, py, bc)
    U = RNG.standard_normal((Nx, Ny))
    C = oracle.unload(xs, px, ys, py, bc, U)
    x = np.sort(RNG.uniform(xs[0], xs[-1], 17))
    y = np.sort(RNG.uniform(ys[0], ys[-1], 13))
    Px, _ = fem_ref.basis_at(xs, px, bc, x)
    Py, _ = fem_ref.basis_at(ys, py, bc, y)
    Lx = fem_ref.legendre_basis_at(xs, px, x)
    Ly = fem_ref.legendre_basis_at(ys, py, y)
    u_fem = Px @ U @ Py.T
    u_leg = Lx @ C @ Ly.T
    assert np.abs(u_fem - u_leg).max() <= 1e-13 * np.abs(u_fem).max()


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_load_of_unload_is_mass(bc):
    """load(unload(U)) = R^T M_P R U R^T M_P R = M_x U M_y (Gram matrix of the
    basis), M from the quadrature reference."""
    xs, px = rand_mesh(4), 5
    ys, py = rand_mesh(3, 0, 1.5), 7
    _, Mx = fem_ref.assemble_quad(xs, px, bc)
    _, My = fem_ref.assemble_quad(ys, py, bc)
    U = RNG.standard_normal((Mx.shape[0], My.shape[0]))
    G = oracle.load(xs, px, ys, py, bc, oracle.unload(xs, px, ys, py, bc, U))
    ref = Mx @ U @ My
    assert np.abs(G - ref).max() <= 1e-13 * np.abs(ref).max()


# ------------------------------------------------- manufactured solution
def _manufactured_error(n, p):
    """u = sin(pi x) sin(pi y) e^{x+y} on [0,1]^2 (north_star); returns the
    L2 error of the ADI solution at eps = 1e-13."""
    pi = math.pi

    def f(x, y):
        e = np.exp(x + y)
        return -e * (2 * (1 - pi * pi) * np.sin(pi * x) * np.sin(pi * y)
                     + 2 * pi * (np.cos(pi * x) * np.sin(pi * y) + np.sin(pi * x) * np.cos(pi * y)))

    def u(x, y):
        return np.sin(pi * x) * np.sin(pi * y) * np.exp(x + y)

    xs = np.linspace(0, 1, n + 1)
    Fleg = W.project_function(xs, p, xs, p, f, nq_extra=30)
    G = oracle.load(xs, p, xs, p, 0, Fleg)
    U, _ = oracle.adi_solve(xs, p, xs, p, 0.0, 0, 1e-13, G)
    x, w = fem_ref.quad_points(xs, p + 12)
    Phi, _ = fem_ref.basis_at(xs, p, 0, x)
    uh = Phi @ U @ Phi.T
    ue = u(x[:, None], x[None, :])
    return math.sqrt(np.einsum("i,j,ij->", w, w, (uh - ue) ** 2))


def test_manufactured_p_convergence():
    """Spectral (exponential) convergence in p at n = 4 for the analytic
    solution, down to the eps = 1e-13 ADI floor: each +2 in p gains >= 400x
    (the h-p FEM rate the paper builds on)."""
    errs = [_manufactured_error(4, p) for p in (2, 4, 6, 8)]
    assert errs[0] < 1e-2
    for a, b in zip(errs, errs[1:]):
        assert a / b >= 400, errs
    assert errs[-1] < 1e-11


@pytest.mark.parametrize("p", [3, 4])
def test_manufactured_h_convergence(p):
    """h-refinement at fixed p: L2 error ratio 2^{p+1} per halving of h
    (within 10%), the optimal rate for degree-p elements."""
    errs = [_manufactured_error(n, p) for n in (2, 4, 8, 16)]
    for a, b in zip(errs[1:], errs[2:]):
        assert a / b == pytest.approx(2.0 ** (p + 1), rel=0.1), errs


def test_l2_norm_is_quadrature():
    """The parity norm tr(U^T M_x U M_y) (Lemma 5.1 norm, reading R12)
    equals the quadrature L2 norm of the FEM function."""
    xs, px = rand_mesh(3), 5
    ys, py = rand_mesh(2), 6
    bc = 1
    U = RNG.standard_normal((oracle.dim(3, px, bc), oracle.dim(2, py, bc)))
    x, wx = fem_ref.quad_points(xs, px + 4)
    y, wy = fem_ref.quad_points(ys, py + 4)
    Px, _ = fem_ref.basis_at(xs, px, bc, x)
    Py, _ = fem_ref.basis_at(ys, py, bc, y)
    uh = Px @ U @ Py.T
    q = np.einsum("i,j,ij->", wx, wy, uh * uh)
    assert oracle.l2_norm_sq(xs, px, ys, py, bc, U) == pytest.approx(q, rel=1e-13)
