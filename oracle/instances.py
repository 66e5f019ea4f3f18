"""TEST INFRASTRUCTURE ONLY: spec string -> synthetic instance.

Specs (all seeded, all built by ``paper_2602_23967_b200.generators``):

    c1:<seed>                 random_qp(2000, 1000, "sparse", density=0.01, seed)   (config 1)
    rqp:<n>:<m>:<kind>:<density>:<seed>   random_qp(...)
    c2:<n>:<m>:<seed>         lasso_style_qp(n, m, seed)                            (config 2 / twins)
    c3:<n>:<k>:<seed>         portfolio_qp(n, k, seed=seed)                         (config 3 / twins)
    c4u:<n>:<seed> / c4i:<n>:<seed>   infeasible_pair(n, seed) [0] / [1]           (config 4)
    c4ur / c4ir                        same on SURVEY.md's random_qp base
    c5:<n>:<w>:<seed>[:diag]  banded_qp(n, n, half_width=w, seed, diagonal_q)       (config 5 / twins)
    qps:<path>                a QPS file read by this repo's reader (io.parse_qps); the
                              reference golden of the same file uses the reference's reader
"""

from __future__ import annotations

from paper_2602_23967_b200 import generators as g


def build(spec: str):
    parts = spec.split(":")
    kind = parts[0]
    if kind == "c1":
        return g.random_qp(2000, 1000, "sparse", density=0.01, seed=int(parts[1]))
    if kind == "rqp":
        n, m, st, dens, seed = parts[1:6]
        return g.random_qp(int(n), int(m), st, density=float(dens), seed=int(seed))
    if kind == "c2":
        return g.lasso_style_qp(int(float(parts[1])), int(float(parts[2])), seed=int(parts[3]))
    if kind == "c3":
        return g.portfolio_qp(int(float(parts[1])), int(parts[2]), seed=int(parts[3]))
    if kind in ("c4u", "c4i", "c4ur", "c4ir"):
        base = "random_qp" if kind.endswith("r") else "diagonal"
        pair = g.infeasible_pair(int(float(parts[1])), seed=int(parts[2]), base=base)
        return pair[0] if kind.startswith("c4u") else pair[1]
    if kind == "qps":
        from paper_2602_23967_b200 import io

        import os

        path = spec.split(":", 1)[1]
        if not os.path.isabs(path):  # relative to the repo root
            path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), path)
        with open(path) as f:
            return io.parse_qps(f.read()).problem
    if kind == "c5":
        diag = len(parts) > 4 and parts[4] == "diag"
        n = int(float(parts[1]))
        return g.banded_qp(n, n, half_width=int(parts[2]), seed=int(parts[3]), diagonal_q=diag)
    raise ValueError(f"unknown instance spec {spec!r}")
