"""Measure the fp64 rounding floor of the ORACLE itself (test infrastructure):
the difference between the oracle's solution and the oracle's solution of the
same problem perturbed at the rounding level (G * (1 + 1e-16 N(0,1)), or every
interior breakpoint scaled by 1 + 2^-52), in three norms:

  *_l2     relative L2(Omega) (Lemma 5.1 mass norm; reading R12)
  *_plain  relative plain coefficient 2-norm ||dU||_F / ||U||_F
  *_max    relative max-abs coefficient difference max|dU| / max|U|

The plain and max-abs floors weight every coefficient alike (the mass norm
de-weights the high-degree bubbles by ~1/k^3), so the GPU parity tests bound
all three (tests/test_gpu_parity.py).  Calls only oracle/ and workloads.py.
Output: tests/golden/oracle_floor.json

    python scripts/oracle_floor.py [config[:iters] ...]

config 5 full takes ~35 CPU-min on 8 cores; `5:16` is the truncated solve
with the first 16 of the J shifts (hpfem_solve_iters), key `config5_iters16`;
`4T` is config 4 solved as the transposed equation (reading R23; the plan's
orientation for config 4), key `config4_T`.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads as W  # noqa: E402


def floor(cfg, iters=-1, transposed=False):
    xs, ys = cfg.breakpoints()
    G = oracle.load(xs, cfg.px, ys, cfg.py, cfg.bc, W.f_leg(cfg, seed=0))
    t = time.time()
    if transposed:  # Alg. 2 on the transposed equation (reading R23): x <-> y, G^T
        bx, by = oracle.split_bc(cfg.bc)
        r, _ = oracle.rounding_floor(ys, cfg.py, xs, cfg.px, cfg.omega, oracle.bc2d(by, bx), cfg.tol,
                                     np.ascontiguousarray(G.T), iters)
    else:
        r, _ = oracle.rounding_floor(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol, G, iters)
    r.update(config=cfg.idx, seconds=time.time() - t, threads=oracle.threads())
    return r


if __name__ == "__main__":
    specs = sys.argv[1:] or ["1", "2", "3", "4", "5"]
    path = os.path.join(ROOT, "tests", "golden", "oracle_floor.json")
    for s in specs:
        c, _, it = s.partition(":")
        tr = c.endswith("T")
        c = c.rstrip("T")
        iters = int(it) if it else -1
        r = floor(W.CONFIGS[int(c)], iters, tr)
        print(s, r, flush=True)
        out = json.load(open(path)) if os.path.exists(path) else {}  # re-read: several runs may share the file
        out[f"config{c}" + (f"_iters{iters}" if it else "") + ("_T" if tr else "")] = r
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
