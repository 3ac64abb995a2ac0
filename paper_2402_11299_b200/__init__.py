"""Thin Python binding of libhpfem_b200.so (the C ABI of include/hpfem.h).

Argument marshalling only: every step of the ADI solve runs in the CUDA
kernels of csrc/kernels.cu.  There is no CPU fallback -- if the extension is
missing or no sm_100 device is usable, calls raise.  PyTorch is used only to
hand over device pointers and the current CUDA stream.

The functions carry the C names (hpfem_plan, hpfem_solve, ...); `Plan` is a
small RAII convenience around them.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPFEM_LIB_PATH") or os.path.join(_HERE, "libhpfem_b200.so")  # override: A/B builds only

HPFEM_BC_DIRICHLET = 0
HPFEM_BC_NEUMANN = 1
HPFEM_BC_DIRICHLET_NEUMANN = 2
HPFEM_BC_NEUMANN_DIRICHLET = 3


def HPFEM_BC_2D(bc_x: int, bc_y: int) -> int:
    """Per-direction 2D boundary code (include/hpfem.h HPFEM_BC_2D)."""
    return 16 + bc_x + 4 * bc_y


HPFEM_OK, HPFEM_EINVAL, HPFEM_ENOTPD, HPFEM_ECUDA, HPFEM_ENOMEM, HPFEM_ENUMERIC = 0, -1, -2, -3, -4, -5
_NAMES = {-1: "EINVAL", -2: "ENOTPD", -3: "ECUDA", -4: "ENOMEM", -5: "ENUMERIC"}

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p
_i, _d = ctypes.c_int, ctypes.c_double
_LIB = None


def _load():
    """Load the CUDA library (lazily, so the build module can be imported
    before it exists).  Missing library = loud ImportError, never a fallback."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2402_11299_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    L.hpfem_plan.argtypes = [_i, _i, _i, _i, _d, _d, _d, _d, _d, _i, _d, _vp, ctypes.POINTER(_vp)]
    L.hpfem_plan_mesh.argtypes = [_dp, _i, _i, _dp, _i, _i, _d, _i, _d, _vp, ctypes.POINTER(_vp)]
    L.hpfem_plan_robin.argtypes = [_dp, _i, _i, _dp, _i, _i, _d, _i, _dp, _d, _vp, ctypes.POINTER(_vp)]
    L.hpfem_plan_info.argtypes = [_vp, _ip, _ip, _ip, _dp, _dp, _dp]
    L.hpfem_plan_shifts.argtypes = [_vp, _dp, _dp]
    L.hpfem_plan_dims.argtypes = [_vp, _ip, _ip, _ip, _ip]
    L.hpfem_plan_path.argtypes = [_vp, _ip, _ip]
    L.hpfem_solve.argtypes = [_vp, _vp, _vp, _vp]
    L.hpfem_solve_iters.argtypes = [_vp, _vp, _vp, _i, _vp]
    L.hpfem_apply.argtypes = [_vp, _vp, _vp, _vp]
    L.hpfem_load.argtypes = [_vp, _vp, _vp, _vp]
    L.hpfem_unload.argtypes = [_vp, _vp, _vp, _vp]
    L.hpfem_solve_batched.argtypes = [_vp, _i, _vp, _vp, _vp]
    L.hpfem_grid.argtypes = [_vp, _dp, _dp]
    L.hpfem_transform.argtypes = [_vp, _vp, _vp, _vp]
    L.hpfem_itransform.argtypes = [_vp, _vp, _vp, _vp]
    L.hpfem_varcoef_apply.argtypes = [_vp, _vp, _vp, _vp, _vp]
    L.hpfem_pcg.argtypes = [_vp, _vp, _vp, _vp, _d, _i, ctypes.POINTER(_i), _dp, _vp]
    L.hpfem_imex_step.argtypes = [_vp, _d, _vp, _vp, _vp]
    L.hpfem_plan1d.argtypes = [_dp, _i, _i, _i, _d, _vp, ctypes.POINTER(_vp)]
    L.hpfem_plan1d_info.argtypes = [_vp, ctypes.POINTER(_i)]
    L.hpfem_solve1d.argtypes = [_vp, _i, _vp, _vp, _vp]
    L.hpfem_plan1d_destroy.argtypes = [_vp]
    L.hpfem_plan_launches.argtypes = [_vp, ctypes.POINTER(ctypes.c_longlong)]
    L.hpfem_plan_profile.argtypes = [_vp, _i]
    L.hpfem_plan_profile_read.argtypes = [_vp, _dp, ctypes.POINTER(ctypes.c_longlong), _dp]
    L.hpfem_plan_destroy.argtypes = [_vp]
    L.hpfem_plan_destroy.restype = None
    L.hpfem_last_error.restype = ctypes.c_char_p
    for f in ("hpfem_plan", "hpfem_plan_mesh", "hpfem_plan_robin", "hpfem_plan_info", "hpfem_plan_dims", "hpfem_plan_path", "hpfem_plan_shifts", "hpfem_solve",
              "hpfem_solve_iters", "hpfem_solve_batched", "hpfem_apply", "hpfem_load", "hpfem_unload", "hpfem_plan_launches", "hpfem_plan_profile",
              "hpfem_plan_profile_read", "hpfem_plan1d", "hpfem_plan1d_info", "hpfem_solve1d", "hpfem_grid",
              "hpfem_transform", "hpfem_itransform", "hpfem_varcoef_apply", "hpfem_pcg", "hpfem_imex_step"):
        getattr(L, f).restype = _i
    _LIB = L
    return L


EXPORTS = ("hpfem_plan", "hpfem_plan_mesh", "hpfem_plan_robin", "hpfem_plan_info", "hpfem_plan_dims", "hpfem_plan_path", "hpfem_plan_shifts", "hpfem_solve",
           "hpfem_solve_iters", "hpfem_solve_batched", "hpfem_apply", "hpfem_load", "hpfem_unload", "hpfem_plan_launches", "hpfem_plan_profile",
           "hpfem_plan_profile_read", "hpfem_plan_destroy", "hpfem_last_error",
           "hpfem_plan1d", "hpfem_plan1d_info", "hpfem_solve1d", "hpfem_plan1d_destroy",
           "hpfem_grid", "hpfem_transform", "hpfem_itransform", "hpfem_varcoef_apply", "hpfem_pcg",
           "hpfem_imex_step")


class HpfemError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"HPFEM_{_NAMES.get(code, code)}: {msg}")
        self.code = code


def hpfem_last_error() -> str:
    return _load().hpfem_last_error().decode()


def _check(rc: int):
    if rc != HPFEM_OK:
        raise HpfemError(rc, hpfem_last_error())


def _ptr(x) -> int:
    """Device pointer of a CUDA float64 contiguous tensor (or a raw int)."""
    if isinstance(x, int):
        return x
    if not x.is_cuda:
        raise ValueError("expected a CUDA tensor (the C ABI takes device pointers)")
    if not x.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    import torch
    if x.dtype != torch.float64:
        raise ValueError("expected float64")
    return x.data_ptr()


def _sized(x, n: int, what: str) -> int:
    """_ptr(x) after checking that the tensor holds exactly n doubles: the C
    ABI takes raw pointers and cannot check sizes, so an undersized buffer
    would be read / written past its end.  Raw ints are passed unchecked."""
    if not isinstance(x, int) and x.numel() != n:
        raise ValueError(f"{what}: expected {n} float64 elements, got {x.numel()} (shape {tuple(x.shape)})")
    return _ptr(x)


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def hpfem_plan(n_x, p_x, n_y, p_y, a, b, c, d, omega, bc, tol, stream=None) -> int:
    h = _vp()
    _check(_load().hpfem_plan(n_x, p_x, n_y, p_y, a, b, c, d, omega, bc, tol, _stream(stream), ctypes.byref(h)))
    return h.value


def hpfem_plan_robin(xs, p_x, ys, p_y, omega, bc, alpha, tol, stream=None) -> int:
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    ys = np.ascontiguousarray(ys, dtype=np.float64)
    al = np.ascontiguousarray(alpha, dtype=np.float64)
    if al.shape != (4,):
        raise ValueError("alpha must hold 4 values (x=a, x=b, y=c, y=d)")
    h = _vp()
    _check(_load().hpfem_plan_robin(xs.ctypes.data_as(_dp), xs.size - 1, p_x, ys.ctypes.data_as(_dp), ys.size - 1,
                                 p_y, omega, bc, al.ctypes.data_as(_dp), tol, _stream(stream), ctypes.byref(h)))
    return h.value


def hpfem_plan_mesh(xs, p_x, ys, p_y, omega, bc, tol, stream=None) -> int:
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    ys = np.ascontiguousarray(ys, dtype=np.float64)
    h = _vp()
    _check(_load().hpfem_plan_mesh(xs.ctypes.data_as(_dp), xs.size - 1, p_x, ys.ctypes.data_as(_dp), ys.size - 1, p_y,
                                omega, bc, tol, _stream(stream), ctypes.byref(h)))
    return h.value


def hpfem_plan_info(plan: int) -> dict:
    Nx, Ny, J = _i(), _i(), _i()
    lx, ly = (ctypes.c_double * 2)(), (ctypes.c_double * 2)()
    g = _d()
    _check(_load().hpfem_plan_info(plan, ctypes.byref(Nx), ctypes.byref(Ny), ctypes.byref(J), lx, ly, ctypes.byref(g)))
    return dict(Nx=Nx.value, Ny=Ny.value, J=J.value, lam_x=np.array(lx[:]), lam_y=np.array(ly[:]), gamma=g.value)


def hpfem_plan_dims(plan: int) -> dict:
    nx, px, ny, py = _i(), _i(), _i(), _i()
    _check(_load().hpfem_plan_dims(plan, ctypes.byref(nx), ctypes.byref(px), ctypes.byref(ny), ctypes.byref(py)))
    return dict(nx=nx.value, px=px.value, ny=ny.value, py=py.value)


def hpfem_plan_path(plan: int) -> dict:
    """{"path": "small" | "tma" | "ldg", "transposed": bool}"""
    path, tr = _i(), _i()
    _check(_load().hpfem_plan_path(plan, ctypes.byref(path), ctypes.byref(tr)))
    return dict(path=("small", "tma", "ldg")[path.value], transposed=bool(tr.value))


def _nn(plan: int) -> int:
    """N_x N_y: elements of a solution / load-space array."""
    i = hpfem_plan_info(plan)
    return i["Nx"] * i["Ny"]


def _nleg(plan: int) -> int:
    """((p_x+1) n_x) ((p_y+1) n_y): elements of a Legendre / grid array."""
    d = hpfem_plan_dims(plan)
    return (d["px"] + 1) * d["nx"] * (d["py"] + 1) * d["ny"]


def hpfem_plan_shifts(plan: int):
    J = hpfem_plan_info(plan)["J"]
    p, q = np.empty(J), np.empty(J)
    _check(_load().hpfem_plan_shifts(plan, p.ctypes.data_as(_dp), q.ctypes.data_as(_dp)))
    return p, q


def hpfem_solve(plan: int, F, U, stream=None):
    n = _nn(plan)
    _check(_load().hpfem_solve(plan, _sized(F, n, "F"), _sized(U, n, "U"), _stream(stream)))


def hpfem_solve_iters(plan: int, F, U, iters: int, stream=None):
    n = _nn(plan)
    _check(_load().hpfem_solve_iters(plan, _sized(F, n, "F"), _sized(U, n, "U"), iters, _stream(stream)))


def hpfem_solve_batched(plan: int, batch: int, F, U, stream=None):
    n = _nn(plan) * max(batch, 0)
    _check(_load().hpfem_solve_batched(plan, batch, _sized(F, n, "F"), _sized(U, n, "U"), _stream(stream)))


def hpfem_plan1d(xs, p: int, bc: int, omega: float, stream=None) -> int:
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    out = _vp()
    _check(_load().hpfem_plan1d(xs.ctypes.data_as(_dp), xs.size - 1, p, bc, omega, _stream(stream), ctypes.byref(out)))
    return out.value


def hpfem_plan1d_info(plan: int) -> int:
    N = _i()
    _check(_load().hpfem_plan1d_info(plan, ctypes.byref(N)))
    return N.value


def hpfem_solve1d(plan: int, nrhs: int, F, U, stream=None):
    n = hpfem_plan1d_info(plan) * max(nrhs, 0)
    _check(_load().hpfem_solve1d(plan, nrhs, _sized(F, n, "F"), _sized(U, n, "U"), _stream(stream)))


def hpfem_plan1d_destroy(plan: int):
    if plan:
        _load().hpfem_plan1d_destroy(plan)


class Plan1D:
    """Batched 1D screened-Poisson solves (K + w^2 M) u = f (the paper's Fig. 1)."""

    def __init__(self, xs, p, bc, omega, stream=None):
        self.handle = hpfem_plan1d(xs, p, bc, omega, stream)
        self.N = hpfem_plan1d_info(self.handle)

    def solve(self, F, U, stream=None):
        """F, U: (nrhs, N) or (N,) device tensors."""
        nrhs = 1 if F.dim() == 1 else int(F.shape[0])
        hpfem_solve1d(self.handle, nrhs, F, U, stream)

    def close(self):
        hpfem_plan1d_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.close()
        except Exception:
            pass


def hpfem_apply(plan: int, U, F, stream=None):
    n = _nn(plan)
    _check(_load().hpfem_apply(plan, _sized(U, n, "U"), _sized(F, n, "F"), _stream(stream)))


def hpfem_load(plan: int, F_leg, G, stream=None):
    _check(_load().hpfem_load(plan, _sized(F_leg, _nleg(plan), "F_leg"), _sized(G, _nn(plan), "G"), _stream(stream)))


def hpfem_unload(plan: int, U, C_leg, stream=None):
    _check(_load().hpfem_unload(plan, _sized(U, _nn(plan), "U"), _sized(C_leg, _nleg(plan), "C_leg"), _stream(stream)))


def hpfem_grid(plan: int, Lx: int, Ly: int):
    """Host grid coordinates (x[(p_x+1) n_x], y[(p_y+1) n_y])."""
    x, y = np.empty(Lx), np.empty(Ly)
    _check(_load().hpfem_grid(plan, x.ctypes.data_as(_dp), y.ctypes.data_as(_dp)))
    return x, y


def hpfem_transform(plan: int, V, C, stream=None):
    n = _nleg(plan)
    _check(_load().hpfem_transform(plan, _sized(V, n, "V"), _sized(C, n, "C"), _stream(stream)))


def hpfem_itransform(plan: int, C, V, stream=None):
    n = _nleg(plan)
    _check(_load().hpfem_itransform(plan, _sized(C, n, "C"), _sized(V, n, "V"), _stream(stream)))


def hpfem_varcoef_apply(plan: int, cgrid, U, F, stream=None):
    n = _nn(plan)
    _check(_load().hpfem_varcoef_apply(plan, _sized(cgrid, _nleg(plan), "cgrid"), _sized(U, n, "U"), _sized(F, n, "F"),
                                       _stream(stream)))


def hpfem_pcg(plan: int, cgrid, G, U, rtol: float, maxit: int, stream=None):
    """Returns (iterations, relative residual)."""
    it, rel = _i(0), _d(0.0)
    n = _nn(plan)
    _check(_load().hpfem_pcg(plan, _sized(cgrid, _nleg(plan), "cgrid"), _sized(G, n, "G"), _sized(U, n, "U"), rtol, maxit,
                             ctypes.byref(it), ctypes.byref(rel), _stream(stream)))
    return it.value, rel.value


def hpfem_imex_step(plan: int, dt: float, U_leg, U_next, stream=None):
    n = _nleg(plan)
    _check(_load().hpfem_imex_step(plan, dt, _sized(U_leg, n, "U_leg"), _sized(U_next, n, "U_next"), _stream(stream)))


def hpfem_plan_launches(plan: int) -> int:
    n = ctypes.c_longlong(0)
    _check(_load().hpfem_plan_launches(plan, ctypes.byref(n)))
    return n.value


KINDS = ("halfstep_bubbles_y", "halfstep_hats_y", "final", "load", "apply", "halfstep_bubbles_x", "halfstep_hats_x")


def hpfem_plan_profile(plan: int, capacity: int):
    _check(_load().hpfem_plan_profile(plan, capacity))


def hpfem_plan_profile_read(plan: int) -> dict:
    ms = (ctypes.c_double * len(KINDS))()
    n = (ctypes.c_longlong * len(KINDS))()
    by = (ctypes.c_double * len(KINDS))()
    _check(_load().hpfem_plan_profile_read(plan, ms, n, by))
    return {k: dict(ms=ms[i], launches=n[i], bytes=by[i]) for i, k in enumerate(KINDS)}


def hpfem_plan_destroy(plan: int):
    if plan:
        _load().hpfem_plan_destroy(plan)


class Plan:
    """RAII wrapper: Plan(xs, px, ys, py, omega, bc, tol) or Plan.uniform(...)."""

    def __init__(self, xs, px, ys, py, omega, bc, tol, stream=None, robin=None):
        if robin is None:
            self.handle = hpfem_plan_mesh(xs, px, ys, py, omega, bc, tol, stream)
        else:
            self.handle = hpfem_plan_robin(xs, px, ys, py, omega, bc, robin, tol, stream)
        info = hpfem_plan_info(self.handle)
        self.__dict__.update(info)
        self.px, self.py, self.bc, self.omega, self.tol = px, py, bc, omega, tol
        self.nx, self.ny = len(xs) - 1, len(ys) - 1

    @classmethod
    def uniform(cls, n_x, p_x, n_y, p_y, a, b, c, d, omega, bc, tol, stream=None):
        obj = cls.__new__(cls)
        obj.handle = hpfem_plan(n_x, p_x, n_y, p_y, a, b, c, d, omega, bc, tol, stream)
        obj.__dict__.update(hpfem_plan_info(obj.handle))
        obj.px, obj.py, obj.bc, obj.omega, obj.tol, obj.nx, obj.ny = p_x, p_y, bc, omega, tol, n_x, n_y
        return obj

    def shifts(self):
        return hpfem_plan_shifts(self.handle)

    def path(self) -> dict:
        return hpfem_plan_path(self.handle)

    def solve(self, F, U, stream=None, iters=None):
        if iters is None:
            hpfem_solve(self.handle, F, U, stream)
        else:
            hpfem_solve_iters(self.handle, F, U, iters, stream)

    def apply(self, U, F, stream=None):
        hpfem_apply(self.handle, U, F, stream)

    def load(self, F_leg, G, stream=None):
        hpfem_load(self.handle, F_leg, G, stream)

    def solve_batched(self, F, U, stream=None):
        """F, U: (batch, Nx, Ny) device tensors."""
        hpfem_solve_batched(self.handle, int(F.shape[0]), F, U, stream)

    def unload(self, U, C_leg, stream=None):
        hpfem_unload(self.handle, U, C_leg, stream)

    def grid(self):
        return hpfem_grid(self.handle, (self.px + 1) * self.nx, (self.py + 1) * self.ny)

    def transform(self, V, C, stream=None):
        hpfem_transform(self.handle, V, C, stream)

    def itransform(self, C, V, stream=None):
        hpfem_itransform(self.handle, C, V, stream)

    def varcoef_apply(self, cgrid, U, F, stream=None):
        hpfem_varcoef_apply(self.handle, cgrid, U, F, stream)

    def pcg(self, cgrid, G, U, rtol=1e-8, maxit=200, stream=None):
        return hpfem_pcg(self.handle, cgrid, G, U, rtol, maxit, stream)

    def imex_step(self, dt, U_leg, U_next, stream=None):
        hpfem_imex_step(self.handle, dt, U_leg, U_next, stream)

    def profile(self, capacity: int):
        hpfem_plan_profile(self.handle, capacity)

    def profile_read(self) -> dict:
        return hpfem_plan_profile_read(self.handle)

    def launches(self) -> int:
        return hpfem_plan_launches(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            hpfem_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
