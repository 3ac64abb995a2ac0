"""The oracle PCG's own fp64 reproducibility floor on the Table 1 cells the
GPU tests use (test infrastructure; calls only oracle/): relative L2 /
plain / max-abs difference between oracle PCG(b) and oracle PCG(b (1 + 1e-16
N(0,1))), seed 5 (reading R24).  Output: tests/golden/pcg_floor.json

    python scripts/pcg_floor.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import oracle.transforms as T  # noqa: E402
from test_gpu_varcoef import GOLDEN, _table1  # noqa: E402  (the test's own inputs)

CELLS = [(1, 8), (1, 16), (2, 8), (2, 32), (3, 16), (3, 64), (3, 128)]

if __name__ == "__main__":
    out = {}
    for m, p in CELLS:
        xs, b, cg = _table1(m, p)
        U1, it1, _ = T.pcg(xs, p, xs, p, 0, cg, b, rtol=GOLDEN["rtol"], tol_pre=GOLDEN["adi_tol"])
        rng = np.random.default_rng(5)
        U2, it2, _ = T.pcg(xs, p, xs, p, 0, cg, b * (1 + 1e-16 * rng.standard_normal(b.shape)), rtol=GOLDEN["rtol"],
                           tol_pre=GOLDEN["adi_tol"])
        d = oracle.rel_diffs(xs, p, xs, p, 0, U2, U1)
        out[f"{m}-{p}"] = dict(G_perturb_l2=d[0], G_perturb_plain=d[1], G_perturb_max=d[2], iters=[it1, it2])
        print(m, p, out[f"{m}-{p}"], flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "pcg_floor.json"), "w") as fh:
        json.dump(out, fh, indent=1)
