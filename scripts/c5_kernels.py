"""Stand-alone hot-kernel timings on one instance under env-knob variants (A/B).

    python scripts/c5_kernels.py [--n 5e7] [--w 5000] [--spec c2] VAR=VAL,VAR=VAL ...  (one arg per variant)

Each variant re-creates the device problem with the knobs set (the knobs are
read at problem/solver creation), then times every hot kernel with the L2
flushed (bench.kernel_table).  Prints one JSON line per variant.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2602_23967_b200 import generators  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=5e7)
    ap.add_argument("--w", type=int, default=5000)
    ap.add_argument("--spec", default="c5")
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    if a.spec == "c5":
        p = generators.banded_qp(int(a.n), int(a.n), half_width=a.w, seed=0)
    elif a.spec == "c2":
        p = generators.lasso_style_qp(1_000_000, 500_000, seed=0)
    elif a.spec == "c3":
        p = generators.portfolio_qp(5_000_000, 100, seed=0)
    else:
        raise SystemExit(a.spec)
    kinds = ("bb_gradient", "bb_step", "p1_At_y", "p2_A_xbar", "x_post", "bb_fold")
    for var in a.variants or [""]:
        saved = {}
        for kv in filter(None, var.split(",")):
            k, v = kv.split("=", 1)
            saved[k] = os.environ.get(k)
            os.environ[k] = v
        out, fixed, per_inner = bench.kernel_table(p, 0, kinds)
        print(json.dumps({"spec": a.spec, "variant": var, **{k: round(v["ms"], 5) for k, v in out.items()},
                          "gbs": {k: round(v["gbs"], 1) for k, v in out.items()}}), flush=True)
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


if __name__ == "__main__":
    main()
