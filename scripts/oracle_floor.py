"""Measure the fp64 rounding floor of the ORACLE itself (test infrastructure):
the relative L2 (Lemma 5.1) difference between the oracle's solution and the
oracle's solution of the same problem perturbed at the rounding level
(G * (1 + 1e-16 N(0,1)), or every interior breakpoint scaled by 1 + 2^-52).
Calls only oracle/ and workloads.py.  Output: tests/golden/oracle_floor.json

    python scripts/oracle_floor.py [config ...]     (config 5 takes ~30 CPU-min on 8 cores)
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


def floor(cfg):
    xs, ys = cfg.breakpoints()
    G = oracle.load(xs, cfg.px, ys, cfg.py, cfg.bc, W.f_leg(cfg, seed=0))
    t = time.time()
    U1, J = oracle.adi_solve(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol, G)
    rng = np.random.default_rng(5)
    U2, _ = oracle.adi_solve(xs, cfg.px, ys, cfg.py, cfg.omega, cfg.bc, cfg.tol,
                             G * (1 + 1e-16 * rng.standard_normal(G.shape)))
    g_l2 = oracle.l2_rel_diff(xs, cfg.px, ys, cfg.py, cfg.bc, U2, U1)
    g_plain = float(np.linalg.norm(U2 - U1) / np.linalg.norm(U1))
    del U2
    xs2, ys2 = xs.copy(), ys.copy()
    xs2[1:-1] *= 1 + 2.0 ** -52
    ys2[1:-1] *= 1 + 2.0 ** -52
    U3, _ = oracle.adi_solve(xs2, cfg.px, ys2, cfg.py, cfg.omega, cfg.bc, cfg.tol, G)
    m_l2 = oracle.l2_rel_diff(xs, cfg.px, ys, cfg.py, cfg.bc, U3, U1)
    m_plain = float(np.linalg.norm(U3 - U1) / np.linalg.norm(U1))
    return dict(config=cfg.idx, J=J, G_perturb_l2=g_l2, G_perturb_plain=g_plain, mesh_ulp_l2=m_l2,
                mesh_ulp_plain=m_plain, seconds=time.time() - t, threads=oracle.threads())


if __name__ == "__main__":
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5]
    path = os.path.join(ROOT, "tests", "golden", "oracle_floor.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for c in cfgs:
        r = floor(W.CONFIGS[c])
        print(r, flush=True)
        out[f"config{c}"] = r
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
