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
from concurrent.futures import ThreadPoolExecutor

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


def _stale(target, deps, flags):
    """Rebuild when the target is missing, older than a dependency, or was
    built with a different command line (the flags -- including the
    HPFEM_NVCC_EXTRA experiment switches -- are stamped next to it)."""
    stamp = target + ".flags"
    if not os.path.exists(target) or not os.path.exists(stamp):
        return True
    if open(stamp).read() != " ".join(flags):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _stamp(target, flags):
    with open(target + ".flags", "w") as fh:
        fh.write(" ".join(flags))


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
               [os.path.join(HERE, "..", "include", "hpfem.h")])
    out = None if verbose else subprocess.DEVNULL
    objs = []
    plan_o = os.path.join(OBJ, "plan.o")
    objs.append(plan_o)
    if force or _stale(plan_o, [os.path.join(CSRC, "plan.cpp")] + headers, CXX_FLAGS):
        subprocess.check_call(["g++", *CXX_FLAGS, "-c", os.path.join(CSRC, "plan.cpp"), "-o", plan_o])
        _stamp(plan_o, CXX_FLAGS)
    jobs = []
    for src, log in (("kernels", "ptxas.log"), ("tma_step", "ptxas_tma.log"), ("solve1d", "ptxas_1d.log"),
                     ("varcoef", "ptxas_vc.log"), ("persist", "ptxas_persist.log")):
        cu = os.path.join(CSRC, src + ".cu")
        if not os.path.exists(cu):
            continue
        obj = os.path.join(OBJ, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [cu] + headers, NVCC_FLAGS):
            jobs.append((cu, obj, os.path.join(OBJ, log)))

    def nvcc(job):
        cu, obj, log = job
        with open(log, "w") as fh:
            subprocess.check_call([NVCC, *NVCC_FLAGS, "-c", cu, "-o", obj], stdout=fh, stderr=subprocess.STDOUT)
        _stamp(obj, NVCC_FLAGS)

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(nvcc, jobs))  # re-raises the first failed compile
    link = ARCH + ["-lquadmath", "-ldl"]  # NVTX3 is header-only (dlopen of the tool's injection library)
    if force or _stale(LIB, objs, link):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-shared", *objs, "-o", tmp, *link], stdout=out)
        os.replace(tmp, LIB)
        _stamp(LIB, link)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
