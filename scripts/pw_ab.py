"""A/B of the C5 norm estimate (100 power iterations, A v and A'w passes) under
ring-path knobs; the estimate must be bitwise the same in every variant.

    python scripts/pw_ab.py "" AQP_RING=0 AQP_RING_OFF=14 ...   (one arg per variant)
"""

from __future__ import annotations

import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_23967_b200 as aq  # noqa: E402
from paper_2602_23967_b200 import engine, generators  # noqa: E402


def main():
    p = generators.banded_qp(50_000_000, 50_000_000, half_width=5000, seed=0)
    v0 = np.random.default_rng(0).standard_normal(p.n)
    for var in sys.argv[1:] or [""]:
        saved = {}
        for kv in filter(None, var.split(",")):
            k, v = kv.split("=", 1)
            saved[k] = os.environ.get(k)
            os.environ[k] = v
        run = engine._Run(p, aq.SolverParams(eps_tol=1e-8), None, 0)
        times = []
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            est, _ann = run.solver.estimate_norm(v0, 100)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t)
        print(json.dumps({"variant": var, "est": est.hex(), "s": [round(x, 4) for x in times],
                          "ring_mask": run.dev.info.ring_mask}), flush=True)
        del run
        gc.collect()
        torch.cuda.empty_cache()
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


if __name__ == "__main__":
    main()
