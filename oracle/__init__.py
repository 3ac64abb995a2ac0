"""ctypes wrapper of the CPU oracle (oracle/hpfem_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2402_11299_b200) never imports it, and this package never imports the
product.  Every function cites the passage of PAPER.md it follows in the C++
source; readings are listed in DESIGN.md.

NEXT-3 (transforms, variable coefficient, PCG) lives in oracle/transforms.py
(numpy), pinned by tests/test_oracle_transforms.py (incl. the paper's
Table 1 iteration counts).

Parity status: every function exported here is pinned by tests/test_oracle_pins.py
against values fixed by the paper or by mathematics (quadrature, dense LAPACK,
mpmath, closed forms); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hpfem_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CFLAGS, "-o", tmp, _SRC, "-lquadmath"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _declare(_lib)
    return _lib


_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_d = ctypes.c_double
_i = ctypes.c_int


def _declare(L):
    L.oracle_last_error.restype = ctypes.c_char_p
    L.oracle_dim.argtypes = [_i, _i, _i]
    L.oracle_threads.restype = _i
    L.oracle_operator_dense.argtypes = [_dp, _i, _i, _i, _d, _d, _dp]
    L.oracle_operator_coo.argtypes = [_dp, _i, _i, _i, _i, _ip, _ip, _dp, _ip]
    L.oracle_factor_dense.argtypes = [_dp, _i, _i, _i, _d, _d, _dp, _ip]
    L.oracle_solve1d.argtypes = [_dp, _i, _i, _i, _d, _d, _dp, _dp, _i]
    L.oracle_spectrum.argtypes = [_dp, _i, _i, _i, _d, _dp]
    L.oracle_shifts.argtypes = [_d, _d, _d, _d, _d, _i, _ip, _dp, _dp, _dp]
    L.oracle_plan.argtypes = [_dp, _i, _i, _dp, _i, _i, _d, _i, _d, _i, _ip, _dp, _dp, _dp, _dp, _dp]
    L.oracle_adi_solve.argtypes = [_dp, _i, _i, _dp, _i, _i, _d, _i, _d, _dp, _dp, _i, _ip]
    L.oracle_apply.argtypes = [_dp, _i, _i, _dp, _i, _i, _d, _i, _dp, _dp]
    L.oracle_load.argtypes = [_dp, _i, _i, _dp, _i, _i, _i, _dp, _dp]
    L.oracle_unload.argtypes = [_dp, _i, _i, _dp, _i, _i, _i, _dp, _dp]
    L.oracle_set_robin.argtypes = [_dp]
    L.oracle_set_robin.restype = None
    L.oracle_set_threads.argtypes = [_i]
    L.oracle_set_threads.restype = None
    for f in ("oracle_operator_dense", "oracle_operator_coo", "oracle_factor_dense", "oracle_solve1d",
              "oracle_spectrum", "oracle_shifts", "oracle_plan", "oracle_adi_solve", "oracle_apply", "oracle_load", "oracle_unload"):
        getattr(L, f).restype = _i


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().oracle_last_error().decode())


def _ptr(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def threads():
    """OpenMP threads used by the oracle's line loops."""
    return lib().oracle_threads()


def set_threads(n: int):
    """OpenMP threads of the line loops (n <= 0: all host cores)."""
    lib().oracle_set_threads(n)


class robin:
    """Context manager: Robin coefficients alpha >= 0 at (x = a, x = b,
    y = c, y = d) for the oracle calls inside the block (the
    1D functions use the first two).  Ends with alpha != 0 must keep their
    hat (a Neumann end of the 1D code)."""

    def __init__(self, alpha4):
        self.a = np.ascontiguousarray(alpha4, dtype=np.float64)

    def __enter__(self):
        lib().oracle_set_robin(_ptr(self.a))
        return self

    def __exit__(self, *exc):
        lib().oracle_set_robin(None)
        return False


def bc2d(bx, by):
    """2D boundary code of per-direction 1D codes (0 Dirichlet, 1 Neumann,
    2 Dirichlet-left / Neumann-right, 3 Neumann-left / Dirichlet-right);
    a plain 0..3 means the same code in both directions."""
    return bx if bx == by else 16 + bx + 4 * by


def split_bc(bc):
    return (bc, bc) if bc < 16 else ((bc - 16) & 3, ((bc - 16) >> 2) & 3)


def dim(n, p, bc):
    return lib().oracle_dim(n, p, bc)


def operator_dense(xs, p, bc, alpha, beta):
    """Dense alpha*K + beta*M of the 1D space (K = -Delta; M)."""
    xs = _f64(xs)
    n = xs.size - 1
    N = dim(n, p, bc)
    out = np.empty((N, N))
    _check(lib().oracle_operator_dense(_ptr(xs), n, p, bc, alpha, beta, _ptr(out)))
    return out


def operator_sparse(xs, p, bc, which):
    """scipy.sparse CSR of K (which=0) or M (which=1)."""
    import scipy.sparse as sp
    xs = _f64(xs)
    n = xs.size - 1
    nnz = ctypes.c_int(0)
    _check(lib().oracle_operator_coo(_ptr(xs), n, p, bc, which, None, None, None, ctypes.byref(nnz)))
    r = np.empty(nnz.value, dtype=np.int32)
    c = np.empty(nnz.value, dtype=np.int32)
    v = np.empty(nnz.value)
    _check(lib().oracle_operator_coo(_ptr(xs), n, p, bc, which, r.ctypes.data_as(_ip), c.ctypes.data_as(_ip),
                                     _ptr(v), ctypes.byref(nnz)))
    N = dim(n, p, bc)
    return sp.csr_matrix((v, (r, c)), shape=(N, N))


def factor_dense(xs, p, bc, alpha, beta):
    """Dense reverse-Cholesky factor L (A = L^T L, Alg. 1)."""
    xs = _f64(xs)
    n = xs.size - 1
    N = dim(n, p, bc)
    out = np.empty((N, N))
    info = (ctypes.c_int * 3)(-1, -1, -1)
    rc = lib().oracle_factor_dense(_ptr(xs), n, p, bc, alpha, beta, _ptr(out), info)
    if rc == -2:
        raise OracleError(rc, f"not positive definite at {tuple(info)}")
    _check(rc)
    return out


def solve1d(xs, p, bc, alpha, beta, f):
    """(alpha K + beta M)^{-1} f for f of shape (N,) or (nrhs, N) (Cor. 4.3)."""
    xs = _f64(xs)
    n = xs.size - 1
    f = _f64(f)
    x = np.empty_like(f)
    nrhs = 1 if f.ndim == 1 else f.shape[0]
    _check(lib().oracle_solve1d(_ptr(xs), n, p, bc, alpha, beta, _ptr(f), _ptr(x), nrhs))
    return x


def spectrum(xs, p, bc, omega):
    """[lambda_min, lambda_max] of the pencil (K + w^2/2 M, M) (reading R4)."""
    xs = _f64(xs)
    lam = np.empty(2)
    _check(lib().oracle_spectrum(_ptr(xs), xs.size - 1, p, bc, omega, _ptr(lam)))
    return lam


def shifts(a, b, c, d, eps, maxJ=4096):
    """(J, gamma, p[J], q[J]) for sigma(A) in [a,b], sigma(B) in [c,d]
    (Alg. 2 lines 2-3; reading R5)."""
    P = np.empty(maxJ)
    Q = np.empty(maxJ)
    J = ctypes.c_int(0)
    g = ctypes.c_double(0)
    _check(lib().oracle_shifts(a, b, c, d, eps, maxJ, ctypes.byref(J), ctypes.byref(g), _ptr(P), _ptr(Q)))
    return J.value, g.value, P[:J.value].copy(), Q[:J.value].copy()


def plan(xs, px, ys, py, omega, bc, tol, maxJ=4096):
    xs, ys = _f64(xs), _f64(ys)
    dims = (ctypes.c_int * 3)()
    lx, ly, P, Q = np.empty(2), np.empty(2), np.empty(maxJ), np.empty(maxJ)
    g = ctypes.c_double(0)
    _check(lib().oracle_plan(_ptr(xs), xs.size - 1, px, _ptr(ys), ys.size - 1, py, omega, bc, tol, maxJ, dims,
                             _ptr(lx), _ptr(ly), ctypes.byref(g), _ptr(P), _ptr(Q)))
    J = dims[2]
    return dict(Nx=dims[0], Ny=dims[1], J=J, lam_x=lx, lam_y=ly, gamma=g.value, p=P[:J].copy(), q=Q[:J].copy())


def adi_solve(xs, px, ys, py, omega, bc, tol, G, iters=-1):
    """Algorithm 2; returns (U, J)."""
    xs, ys, G = _f64(xs), _f64(ys), _f64(G)
    U = np.empty_like(G)
    J = ctypes.c_int(0)
    _check(lib().oracle_adi_solve(_ptr(xs), xs.size - 1, px, _ptr(ys), ys.size - 1, py, omega, bc, tol, _ptr(G),
                                  _ptr(U), iters, ctypes.byref(J)))
    return U, J.value


def apply(xs, px, ys, py, omega, bc, U):
    """A_x U M_y + M_x U A_y (eq. adi:poisson)."""
    xs, ys, U = _f64(xs), _f64(ys), _f64(U)
    F = np.empty_like(U)
    _check(lib().oracle_apply(_ptr(xs), xs.size - 1, px, _ptr(ys), ys.size - 1, py, omega, bc, _ptr(U), _ptr(F)))
    return F


def load(xs, px, ys, py, bc, Fleg):
    """G = R_x^T M_P,x F_leg M_P,y R_y."""
    xs, ys, Fleg = _f64(xs), _f64(ys), _f64(Fleg)
    bx, by = split_bc(bc)
    Nx, Ny = dim(xs.size - 1, px, bx), dim(ys.size - 1, py, by)
    G = np.empty((Nx, Ny))
    _check(lib().oracle_load(_ptr(xs), xs.size - 1, px, _ptr(ys), ys.size - 1, py, bc, _ptr(Fleg), _ptr(G)))
    return G


def unload(xs, px, ys, py, bc, U):
    """C_leg = R_x U R_y^T: piecewise-Legendre coefficients of the FEM function
    (NEXT-1 of SURVEY 8(f); basis change of P:L392-L399 / eq. app:1 P:L1074)."""
    xs, ys, U = _f64(xs), _f64(ys), _f64(U)
    Lx, Ly = (px + 1) * (xs.size - 1), (py + 1) * (ys.size - 1)
    C = np.empty((Lx, Ly))
    _check(lib().oracle_unload(_ptr(xs), xs.size - 1, px, _ptr(ys), ys.size - 1, py, bc, _ptr(U), _ptr(C)))
    return C


def l2_norm_sq(xs, px, ys, py, bc, U):
    """||u||^2_{L2} of the FEM function with coefficients U: tr(U^T M_x U M_y)
    = ||V U L^T||_F^2 for M_x = V^T V, M_y = L^T L (the Lemma 5.1 norm,
    P:L733).  Used as the parity norm (reading R12)."""
    bx, by = split_bc(bc)
    Mx = operator_sparse(xs, px, bx, 1)
    My = operator_sparse(ys, py, by, 1)
    U = _f64(U)
    A = Mx @ U
    B = (My @ U.T).T
    return float(np.einsum("ij,ij->", A, B))


def l2_rel_diff(xs, px, ys, py, bc, U, Uref):
    """||u - u_ref||_{L2} / ||u_ref||_{L2}."""
    d = l2_norm_sq(xs, px, ys, py, bc, np.asarray(U) - np.asarray(Uref))
    r = l2_norm_sq(xs, px, ys, py, bc, Uref)
    return float(np.sqrt(max(d, 0.0) / r))


def rel_diffs(xs, px, ys, py, bc, U, Uref):
    """(L2(Omega) relative, plain coefficient 2-norm relative, max-abs
    relative) differences of two coefficient arrays: the three parity
    measures (reading R12; the last two weight every coefficient alike)."""
    U, Uref = np.asarray(U), np.asarray(Uref)
    d = U - Uref
    nr = np.linalg.norm(Uref)
    mr = np.abs(Uref).max() if Uref.size else 0.0
    return (l2_rel_diff(xs, px, ys, py, bc, U, Uref) if nr > 0 else float(np.linalg.norm(d)),
            float(np.linalg.norm(d) / nr) if nr > 0 else float(np.linalg.norm(d)),
            float(np.abs(d).max() / mr) if mr > 0 else float(np.abs(d).max(initial=0.0)))


def w_rel_diff(ys, py, bc, U, Uref):
    """Relative plain 2-norm difference of W = U M_y, the ADI iterate of
    Alg. 2 before the final W_J C^{-1} (C = M_y, reading R6):
    ||(U - Uref) M_y||_F / ||Uref M_y||_F.  The mass solve M_y^{-1} amplifies
    rounding by up to kappa(M_y) (~1e16 on config 5's graded mesh), so a
    truncated iterate is compared here, where that amplification is undone."""
    _, by = split_bc(bc)
    My = operator_sparse(ys, py, by, 1)
    U, Uref = np.asarray(U), np.asarray(Uref)
    Wr = (My @ Uref.T).T
    Wd = (My @ (U - Uref).T).T
    return float(np.linalg.norm(Wd) / np.linalg.norm(Wr)) if np.any(Wr) else float(np.linalg.norm(Wd))


def rounding_floor(xs, px, ys, py, omega, bc, tol, G, iters=-1, robin_alpha=None):
    """The oracle's own fp64 reproducibility floor for one problem: the
    rel_diffs between adi_solve(G) and adi_solve of the same problem
    perturbed at the rounding level -- G * (1 + 1e-16 N(0,1)) (seed 5), and
    every interior breakpoint scaled by 1 + 2^-52.  Two correct fp64
    implementations of Algorithm 2 that round differently cannot be expected
    to agree better than this.  robin_alpha: the solves run
    with those Robin coefficients (the norms -- mass matrices only -- do not
    depend on them).  Returns (dict of the *_l2 / *_plain / *_max / *_w
    floors of both perturbations, the unperturbed solution)."""
    G = _f64(G)
    xs2, ys2 = np.array(xs, dtype=np.float64), np.array(ys, dtype=np.float64)
    xs2[1:-1] *= 1 + 2.0 ** -52
    ys2[1:-1] *= 1 + 2.0 ** -52
    rng = np.random.default_rng(5)
    Gp = G * (1 + 1e-16 * rng.standard_normal(G.shape))

    def solves():
        U1, J = adi_solve(xs, px, ys, py, omega, bc, tol, G, iters)
        U2, _ = adi_solve(xs, px, ys, py, omega, bc, tol, Gp, iters)
        U3, _ = adi_solve(xs2, px, ys2, py, omega, bc, tol, G, iters)
        return U1, U2, U3, J

    if robin_alpha is None:
        U1, U2, U3, J = solves()
    else:
        with robin(robin_alpha):
            U1, U2, U3, J = solves()
    g = rel_diffs(xs, px, ys, py, bc, U2, U1) + (w_rel_diff(ys, py, bc, U2, U1),)
    m = rel_diffs(xs, px, ys, py, bc, U3, U1) + (w_rel_diff(ys, py, bc, U3, U1),)
    return dict(J=J, iters=iters, G_perturb_l2=g[0], G_perturb_plain=g[1], G_perturb_max=g[2], G_perturb_w=g[3],
                mesh_ulp_l2=m[0], mesh_ulp_plain=m[1], mesh_ulp_max=m[2], mesh_ulp_w=m[3]), U1
