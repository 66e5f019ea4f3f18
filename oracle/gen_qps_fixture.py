"""TEST INFRASTRUCTURE ONLY: write the QPS fixture of the real-instance parity test.

    python oracle/gen_qps_fixture.py tests/golden/qps_mixed_400.qps

A deterministic, feasible and bounded QP written as QPS text that exercises
every convention of the reference reader (anchorqp/qps.py:1-16, 43-290):
L / G / E rows with RANGES (R > 0 and R < 0 on E rows, L and G rows), free N
rows beyond the objective, an RHS entry on the objective row (the objective
constant), UP with a negative value on an untouched lower bound, MI / PL /
FX / FR / LO / UP bounds, and a QMATRIX section listing both triangles.
The golden solve of this file by the reference (its own parser) is recorded
with ``oracle/run_reference.py qps:<path>``.
"""

from __future__ import annotations

import sys

import numpy as np


def build(n: int = 400, m: int = 200, seed: int = 3) -> str:
    rng = np.random.default_rng(seed)
    cols = [f"x{j}" for j in range(n)]
    xs = rng.uniform(-1.0, 1.0, n)  # a feasible point
    # A: ~6 entries per row
    rows = []
    for i in range(m):
        js = np.sort(rng.choice(n, 6, replace=False))
        rows.append((js, np.round(rng.normal(size=6), 6)))
    ax = np.array([v @ xs[js] for js, v in rows])
    kinds = rng.choice(["L", "G", "E"], m, p=[0.4, 0.4, 0.2])
    rhs, rng_vals = {}, {}
    for i, k in enumerate(kinds):
        slack = round(float(rng.uniform(0.1, 1.0)), 6)
        if k == "L":
            rhs[i] = round(ax[i] + slack, 6)
        elif k == "G":
            rhs[i] = round(ax[i] - slack, 6)
        else:
            rhs[i] = round(ax[i], 6)
        if i % 5 == 0:  # RANGES: L [r-|R|, r], G [r, r+|R|], E sign-dependent
            R = round(float(rng.uniform(0.5, 2.0)), 6) * (-1.0 if (k == "E" and i % 10 == 0) else 1.0)
            if k == "E" and R < 0:
                rhs[i] = round(ax[i] + 0.25, 6)  # [r + R, r] must hold A x*
            if k == "E" and R > 0:
                rhs[i] = round(ax[i] - 0.25, 6)  # [r, r + R]
            rng_vals[i] = R
    # Q: diagonal + sparse symmetric couplings, PSD by diagonal dominance
    pairs = {}
    for _ in range(3 * n):
        a, b = rng.integers(0, n, 2)
        if a != b:
            pairs[(min(a, b), max(a, b))] = round(float(rng.normal()) * 0.3, 6)
    deg = np.zeros(n)
    for (a, b), v in pairs.items():
        deg[a] += abs(v)
        deg[b] += abs(v)
    diag = np.round(deg + rng.uniform(0.1, 1.0, n), 6)
    cost = np.round(rng.normal(size=n), 6)

    out = ["* QPS fixture: every reader convention (oracle/gen_qps_fixture.py)", "NAME          MIXED400", "ROWS",
           " N  obj"]
    out += [f" {k}  r{i}" for i, k in enumerate(kinds)]
    out += [" N  free1", " N  free2"]
    out.append("COLUMNS")
    col_entries = {j: [] for j in range(n)}
    for i, (js, v) in enumerate(rows):
        for j, a in zip(js, v):
            col_entries[j].append((f"r{i}", a))
    for j in range(n):
        ent = [("obj", cost[j])] if cost[j] != 0 else []
        ent += col_entries[j]
        if j % 7 == 0:
            ent.append(("free1", 1.5))
        if j % 11 == 0:
            ent.append(("free2", -2.0))
        for a in range(0, len(ent), 2):
            chunk = ent[a:a + 2]
            out.append("    " + cols[j] + "  " + "  ".join(f"{r}  {format(float(v), '.17g')}" for r, v in chunk))
    out.append("RHS")
    out.append(f"    RHS  obj  {-12.5}")  # objective constant 12.5
    for i in range(m):
        out.append(f"    RHS  r{i}  {format(float(rhs[i]), '.17g')}")
    out.append("RANGES")
    for i, R in rng_vals.items():
        out.append(f"    RNG  r{i}  {format(float(R), '.17g')}")
    out.append("BOUNDS")
    for j in range(n):
        lo, hi = xs[j] - 1.0, xs[j] + 1.0
        c = j % 8
        if c == 0:
            out.append(f" FR BND  {cols[j]}")
        elif c == 1:
            out.append(f" MI BND  {cols[j]}")
            out.append(f" UP BND  {cols[j]}  {format(round(hi, 6), '.17g')}")
        elif c == 2:
            out.append(f" LO BND  {cols[j]}  {format(round(lo, 6), '.17g')}")
            out.append(f" UP BND  {cols[j]}  {format(round(hi, 6), '.17g')}")
        elif c == 3:
            out.append(f" LO BND  {cols[j]}  {format(round(lo, 6), '.17g')}")
            out.append(f" PL BND  {cols[j]}")
        elif c == 4 and xs[j] < -0.2:  # negative UP on an untouched lower bound: lower drops to -inf
            out.append(f" UP BND  {cols[j]}  {format(round(xs[j] + 0.1, 6), '.17g')}")
        elif c == 4:
            out.append(f" MI BND  {cols[j]}")
        elif c == 5:
            out.append(f" FX BND  {cols[j]}  {format(round(float(xs[j]), 6), '.17g')}")
        # c = 6, 7: free of BOUNDS entries except the default [0, inf) when x* >= 0
        elif xs[j] < 0:
            out.append(f" FR BND  {cols[j]}")
    out.append("QMATRIX")
    qent = [(j, j, diag[j]) for j in range(n)] + [(a, b, v) for (a, b), v in pairs.items()] + \
        [(b, a, v) for (a, b), v in pairs.items()]
    qent.sort()
    for a, b, v in qent:
        out.append(f"    {cols[a]}  {cols[b]}  {format(float(v), '.17g')}")
    out.append("ENDATA")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    with open(sys.argv[1], "w") as f:
        f.write(build())
