"""TEST INFRASTRUCTURE ONLY -- never imported by the product package.

Bridges instances between this repo's types and the real reference package
(``anchorqp``, built by ``oracle/build_ref.sh`` into ``oracle/_ref``).  Used by
the golden-fixture script, the parity tests and bench.py's reference arm.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def load_reference():
    """Import the built reference ``anchorqp`` (Cython backend) or return None."""
    if not os.path.isdir(os.path.join(REF_DIR, "anchorqp")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import anchorqp  # noqa: E402

    return anchorqp


def to_reference(problem, aq):
    """Rebuild one of our QpProblem objects as a reference ``anchorqp.QpProblem``
    (identical arrays; the reference re-validates them)."""

    def mat(s):
        return aq.SparseMatrix(s.rows, s.cols, s.indptr, s.indices, s.data)

    q = problem.quad
    if q.kind == "diagonal":
        rq = aq.DiagonalQuad(q.values)
    elif q.kind == "sparse":
        rq = aq.SparseQuad(mat(q.upper), q.diag)
    else:
        rq = aq.SparseLowRankQuad(aq.SparseQuad(mat(q.p.upper), q.p.diag), mat(q.r))
    return aq.QpProblem(
        quad=rq,
        cost=problem.cost,
        constraint_matrix=mat(problem.constraint_matrix),
        var_bounds=aq.Bounds(problem.var_bounds.lower, problem.var_bounds.upper),
        con_bounds=aq.Bounds(problem.con_bounds.lower, problem.con_bounds.upper),
        name=problem.name,
    )
