"""Phase breakdown of one C5 solve call from host arrays (where the e2e time goes).

    python scripts/e2e_phases.py [n] [half_width] [iters]
"""

from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2602_23967_b200 as aq  # noqa: E402
from paper_2602_23967_b200 import generators  # noqa: E402


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 50_000_000
    w = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    t = time.perf_counter()
    p = generators.banded_qp(n, n, half_width=w, seed=0)
    out = {"gen_s": time.perf_counter() - t}
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    torch.cuda.synchronize()

    def ph(name, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        out[name] = time.perf_counter() - t0
        return r

    params = aq.SolverParams(eps_tol=1e-8, iter_limit=iters)
    os.environ["AQP_PHASES"] = "1"  # engine / device print their phase split to stderr
    res = ph("solve_total", lambda: aq.solve(p, params))
    out["inner"] = res.inner_iterations
    out["e2e_inner_per_s"] = res.inner_iterations / out["solve_total"]
    ph("solve_total_again", lambda: aq.solve(p, params))  # warm: context and pools exist
    out["n"] = n
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
