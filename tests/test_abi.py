"""CPU-side checks of the C ABI library (no compute calls without a GPU):
it builds, loads, exports every symbol include/hpfem.h declares, shares no
code with the oracle, and refuses to run without a device (no fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hpfem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hpfem_[a-z0-9_]+)\s*\(", src)))


def _lib_path():
    import importlib.util

    spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2402_11299_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


def test_library_exports_every_declared_symbol():
    lib = _lib_path()
    names = _declared()
    assert len(names) >= 12
    L = ctypes.CDLL(lib)
    for n in names:
        assert hasattr(L, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    assert "oracle_" not in nm


def test_binding_names_match_header():
    import paper_2402_11299_b200 as hp

    for n in _declared():
        assert n in hp.EXPORTS and callable(getattr(hp, n)), n


def test_no_shared_code_with_oracle():
    """The product sources never include / import the oracle, and vice versa."""
    prod = os.path.join(ROOT, "paper_2402_11299_b200")
    for dp, _, fs in os.walk(prod):
        for f in fs:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                s = open(os.path.join(dp, f)).read()
                for bad in ("import oracle", "from oracle", "hpfem_oracle", "liboracle"):
                    assert bad not in s, (f, bad)
    for f in ("hpfem_oracle.cpp", "__init__.py"):
        s = open(os.path.join(ROOT, "oracle", f)).read()
        for bad in ("ops1d.h", "hpfem_internal", "import paper_2402_11299_b200", "from paper_2402_11299_b200",
                    "libhpfem_b200"):
            assert bad not in s, (f, bad)


def test_refuses_without_device():
    """No GPU here: hpfem_plan must fail with HPFEM_ECUDA, never compute on
    the CPU."""
    import torch

    if torch.cuda.is_available():
        return
    L = ctypes.CDLL(_lib_path())
    L.hpfem_plan_mesh.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    xs = np.linspace(0, 1, 3)
    h = ctypes.c_void_p()
    p = xs.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    rc = L.hpfem_plan_mesh(p, 2, 4, p, 2, 4, 0.0, 0, 1e-10, None, ctypes.byref(h))
    assert rc == -3  # HPFEM_ECUDA
    rc = L.hpfem_plan_mesh(p, 2, 1, p, 2, 4, 0.0, 0, 1e-10, None, ctypes.byref(h))
    assert rc == -1  # HPFEM_EINVAL is checked before touching the device


def test_boundary_codes_validated_before_device():
    """Boundary codes (include/hpfem.h): 0..3 and HPFEM_BC_2D(0..3, 0..3) are
    accepted (-> ECUDA here, no device); anything else, or a Neumann-only
    direction with w = 0, is EINVAL before the device is touched."""
    import paper_2402_11299_b200 as hp

    L = ctypes.CDLL(_lib_path())
    L.hpfem_plan_mesh.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    xs = np.linspace(0, 1, 3)
    h = ctypes.c_void_p()
    p = xs.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    ok = -3 if not __import__("torch").cuda.is_available() else 0

    def rc(bc, om):
        r = L.hpfem_plan_mesh(p, 2, 4, p, 2, 4, om, bc, 1e-10, None, ctypes.byref(h))
        if r == 0:
            ctypes.CDLL(_lib_path()).hpfem_plan_destroy(h)
        return r

    for bc in (0, 2, 3, hp.HPFEM_BC_2D(2, 3), hp.HPFEM_BC_2D(0, 2)):
        assert rc(bc, 0.0) == ok, bc
    for bc in (1, hp.HPFEM_BC_2D(1, 1), hp.HPFEM_BC_2D(3, 1)):
        assert rc(bc, 1.0) == ok, bc
        assert rc(bc, 0.0) == -1, bc  # a Neumann-only direction needs w != 0
    for bc in (-1, 4, 15, 32, hp.HPFEM_BC_2D(0, 4)):
        assert rc(bc, 1.0) == -1, bc


def test_binding_checks_sizes():
    """The binding refuses a buffer of the wrong size before the C ABI sees
    the raw pointer (an undersized buffer would be read / written past its
    end).  No device needed: the size check comes first."""
    import pytest
    import torch

    import paper_2402_11299_b200 as hp

    with pytest.raises(ValueError):
        hp._sized(torch.zeros(3, dtype=torch.float64), 4, "F")
    assert hp._sized(12345, 4, "F") == 12345  # raw pointers pass unchecked
