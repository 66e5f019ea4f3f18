"""Power-iteration kernels of one C5 estimate_norm (for an ncu launch list):

    ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none \
        python scripts/pw_kernels.py [n] [iters]
"""

from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_23967_b200 as aq  # noqa: E402
from paper_2602_23967_b200 import engine, generators  # noqa: E402


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 50_000_000
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    p = generators.banded_qp(n, n, half_width=5000, seed=0)
    params = aq.SolverParams(eps_tol=1e-8)
    run = engine._Run(p, params, None, 0)
    v0 = np.random.default_rng(0).standard_normal(p.n)
    for reps in (1, 2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        est, ann = run.solver.estimate_norm(v0, iters)
        torch.cuda.synchronize()
        print(f"estimate_norm iters={iters} est={est!r} {time.perf_counter() - t:.4f}s", flush=True)


if __name__ == "__main__":
    main()
