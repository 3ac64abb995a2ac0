"""Compile the in-tree shared library libhpfem_b200.so for sm_100a.

  g++  -O2 -std=gnu++17   csrc/plan.cpp     (host plan, binary128 shifts)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo  csrc/kernels.cu, tma_step.cu, solve1d.cu, varcoef.cu
  nvcc -shared ... -lquadmath  ->  paper_2402_11299_b200/libhpfem_b200.so

nvcc cross-compiles without a GPU, so this runs on the CPU build box too.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libhpfem_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"] + \
    os.environ.get("HPFEM_NVCC_EXTRA", "").split()  # experiments only
CXX_FLAGS = ["-O2", "-std=gnu++17", "-fPIC", "-Wall", "-Wextra", f"-I{CUDA}/include"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(HERE, "..", "include", "hpfem.h")]
    plan_o = os.path.join(OBJ, "plan.o")
    kern_o = os.path.join(OBJ, "kernels.o")
    tma_o = os.path.join(OBJ, "tma_step.o")
    s1d_o = os.path.join(OBJ, "solve1d.o")
    vc_o = os.path.join(OBJ, "varcoef.o")
    out = None if verbose else subprocess.DEVNULL
    if force or _stale(plan_o, [os.path.join(CSRC, "plan.cpp")] + headers):
        subprocess.check_call(["g++", *CXX_FLAGS, "-c", os.path.join(CSRC, "plan.cpp"), "-o", plan_o])
    if force or _stale(kern_o, [os.path.join(CSRC, "kernels.cu")] + headers):
        log = os.path.join(OBJ, "ptxas.log")
        with open(log, "w") as fh:
            subprocess.check_call([NVCC, *NVCC_FLAGS, "-c", os.path.join(CSRC, "kernels.cu"), "-o", kern_o],
                                  stdout=fh, stderr=subprocess.STDOUT)
    if force or _stale(tma_o, [os.path.join(CSRC, "tma_step.cu")] + headers):
        log = os.path.join(OBJ, "ptxas_tma.log")
        with open(log, "w") as fh:
            subprocess.check_call([NVCC, *NVCC_FLAGS, "-c", os.path.join(CSRC, "tma_step.cu"), "-o", tma_o],
                                  stdout=fh, stderr=subprocess.STDOUT)
    if force or _stale(s1d_o, [os.path.join(CSRC, "solve1d.cu")] + headers):
        log = os.path.join(OBJ, "ptxas_1d.log")
        with open(log, "w") as fh:
            subprocess.check_call([NVCC, *NVCC_FLAGS, "-c", os.path.join(CSRC, "solve1d.cu"), "-o", s1d_o],
                                  stdout=fh, stderr=subprocess.STDOUT)
    if force or _stale(vc_o, [os.path.join(CSRC, "varcoef.cu")] + headers):
        log = os.path.join(OBJ, "ptxas_vc.log")
        with open(log, "w") as fh:
            subprocess.check_call([NVCC, *NVCC_FLAGS, "-c", os.path.join(CSRC, "varcoef.cu"), "-o", vc_o],
                                  stdout=fh, stderr=subprocess.STDOUT)
    if force or _stale(LIB, [plan_o, kern_o, tma_o, s1d_o, vc_o]):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-shared", *ARCH, plan_o, kern_o, tma_o, s1d_o, vc_o, "-o", tmp, "-lquadmath"],
                              stdout=out)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
