"""CPU: instance files (paper_2602_23967_b200.io) -- the binary format round
trip, and parity with the reference's own JSON and QPS readers/writers
(``aq/serialize.py``, ``aq/qps.py``) run from oracle/_ref."""

import os

import numpy as np
import pytest

import instances
import refbridge
from paper_2602_23967_b200 import io as aqio
from paper_2602_23967_b200.errors import ParseError, UnsupportedSection

AQ = refbridge.load_reference()
needs_ref = pytest.mark.skipif(AQ is None, reason="oracle/_ref (reference build) missing")

SPECS = ["rqp:40:25:sparse:0.2:3", "rqp:30:20:diagonal:0.3:4", "rqp:20:12:low_rank:0.3:5", "c1:2",
         "c4i:1e3:1", "c3:2e3:100:0"]


def same_problem(p, q):
    assert p.n == q.n and p.m == q.m
    a, b = p.constraint_matrix, q.constraint_matrix
    np.testing.assert_array_equal(a.indptr, b.indptr)
    np.testing.assert_array_equal(a.indices, b.indices)
    np.testing.assert_array_equal(a.data, b.data)
    np.testing.assert_array_equal(p.cost, q.cost)
    for x, y in ((p.var_bounds, q.var_bounds), (p.con_bounds, q.con_bounds)):
        np.testing.assert_array_equal(x.lower, y.lower)
        np.testing.assert_array_equal(x.upper, y.upper)
    qa, qb = p.quad, q.quad
    assert type(qa).__name__ == type(qb).__name__
    if hasattr(qa, "values"):
        np.testing.assert_array_equal(qa.values, qb.values)
    else:
        ua = qa.upper if hasattr(qa, "upper") else qa.p.upper
        ub = qb.upper if hasattr(qb, "upper") else qb.p.upper
        np.testing.assert_array_equal(ua.indptr, ub.indptr)
        np.testing.assert_array_equal(ua.indices, ub.indices)
        np.testing.assert_array_equal(ua.data, ub.data)
        if hasattr(qa, "r"):
            np.testing.assert_array_equal(qa.r.data, qb.r.data)
            np.testing.assert_array_equal(qa.r.indices, qb.r.indices)


@pytest.mark.parametrize("spec", SPECS)
def test_binary_round_trip(tmp_path, spec):
    p = instances.build(spec)
    f = tmp_path / "x.aqpz"
    aqio.save_problem(p, f)
    same_problem(p, aqio.load_problem(f))


def test_binary_rejects_garbage(tmp_path):
    f = tmp_path / "bad.aqpz"
    f.write_bytes(b"not an npz")
    with pytest.raises(ParseError):
        aqio.load_problem(f)


@needs_ref
@pytest.mark.parametrize("spec", SPECS)
def test_json_documents_match_reference(tmp_path, spec):
    p = instances.build(spec)
    rp = refbridge.to_reference(p, AQ)
    from anchorqp import serialize as rser

    ours, theirs = tmp_path / "ours.json", tmp_path / "theirs.json"
    aqio.dump_problem_json(p, ours)
    rser.dump_problem(rp, theirs)
    assert aqio.problem_to_dict(p) == rser.problem_to_dict(rp)
    same_problem(p, aqio.load_problem(theirs))       # reference document -> ours
    back = rser.load_problem_json(ours)               # our document -> reference
    same_problem(p, back)


HAND_QPS = [
    # ranges on every row type, set names present / absent, objective constant
    """NAME TESTQP
ROWS
 N  COST
 L  LIM1
 G  LIM2
 E  MYEQN
 E  NEGRNG
 N  FREE1
COLUMNS
    X1  COST  1.0  LIM1  1.0
    X1  LIM2  1.0
    X2  COST  2.0  LIM1  1.0
    X2  MYEQN  -1.0  NEGRNG 3.5
    X3  COST  -1.0  FREE1  2.0
    X3  MYEQN  1.0
RHS
    RHS  COST  -4.5
    RHS  LIM1  4.0  LIM2  1.0
    MYEQN  7.0
    RHS  NEGRNG  2.0
RANGES
    RNG  LIM1  2.5  LIM2  -3.0
    RNG  MYEQN  1.5  NEGRNG  -0.5
BOUNDS
 UP BND  X1  4.0
 LO BND  X2  -1.0
 UP BND  X2  1.0
 MI BND  X3
 UP BND  X3  -2.0
 UP BND  X4  -1.0
 FR BND  X5
 PL BND  X1
 FX BND  X6  0.25
QUADOBJ
    X1  X1  2.0
    X1  X2  -0.5
    X2  X2  3.0
    X3  X3  1.0
ENDATA
""",
    # QMATRIX listing both triangles, free-format, comment lines, no ENDATA
    """* a comment
NAME
 QM
ROWS
 N obj
 E c1
COLUMNS
 x obj 1 c1 1
 y obj -1 c1 1
RHS
 rhs c1 1
QMATRIX
 x x 4
 x y 1
 y x 1
 y y 2
""",
    # diagonal-only quadratic section becomes a DiagonalQuad
    """NAME DIAG
ROWS
 N OBJ
 G R1
COLUMNS
 A OBJ 1 R1 2
 B R1 1
QUADOBJ
 A A 1.5
 B B 0.5
ENDATA
""",
]


@needs_ref
@pytest.mark.parametrize("k", range(len(HAND_QPS)))
def test_qps_parse_matches_reference(k):
    from anchorqp import qps as rq

    ours, theirs = aqio.parse_qps(HAND_QPS[k], name="t"), rq.parse_qps(HAND_QPS[k], name="t")
    assert ours.objective_constant == theirs.objective_constant
    assert ours.problem.name == theirs.problem.name
    same_problem(ours.problem, theirs.problem)


@needs_ref
@pytest.mark.parametrize("spec", ["rqp:40:25:sparse:0.2:3", "rqp:30:20:diagonal:0.3:4", "c4u:1e3:1"])
def test_qps_write_parse_round_trip_and_cross(spec):
    from anchorqp import qps as rq

    p = instances.build(spec)
    rp = refbridge.to_reference(p, AQ)
    text = aqio.write_qps(p, objective_constant=1.25)
    doc = aqio.parse_qps(text)
    assert doc.objective_constant == 1.25
    # a ranged row travels as (upper, upper - lower): its lower bound comes
    # back within an ulp (the reference's convention, aq/qps.py:200-210)
    np.testing.assert_allclose(doc.problem.con_bounds.lower, p.con_bounds.lower, rtol=1e-15, atol=1e-15)
    np.testing.assert_array_equal(doc.problem.con_bounds.upper, p.con_bounds.upper)
    same_problem(doc.problem, rq.parse_qps(text).problem)       # the reference reads our text identically
    theirs = rq.write_qps(rp, 1.25)
    same_problem(aqio.parse_qps(theirs).problem, rq.parse_qps(theirs).problem)  # and we read theirs


BAD_QPS = [
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n    MARKER 'MARKER' 'INTORG'\nENDATA\n", UnsupportedSection),
    ("NAME X\nFOO\nENDATA\n", UnsupportedSection),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1\nBOUNDS\n BV BND X\nENDATA\n", UnsupportedSection),
    ("NAME X\nOBJSENSE\n MAX\nENDATA\n", UnsupportedSection),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X R9 1\nENDATA\n", ParseError),
    ("NAME X\nROWS\n L R1\nCOLUMNS\n X R1 1\nENDATA\n", ParseError),
    ("NAME X\nROWS\n N OBJ\n N OBJ\nENDATA\n", ParseError),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ abc\nENDATA\n", ParseError),
    ("  X OBJ 1\n", ParseError),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1\nQUADOBJ\n X X\nENDATA\n", ParseError),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1\nBOUNDS\n ZZ BND X 1\nENDATA\n", ParseError),
]


@needs_ref
@pytest.mark.parametrize("k", range(len(BAD_QPS)))
def test_qps_errors_match_reference(k):
    from anchorqp import qps as rq
    from anchorqp import errors as rerr

    text, exc = BAD_QPS[k]
    with pytest.raises(exc) as ours:
        aqio.parse_qps(text)
    with pytest.raises(rerr.ParseError) as theirs:
        rq.parse_qps(text)
    assert isinstance(theirs.value, rerr.UnsupportedSection) == isinstance(ours.value, UnsupportedSection)
    assert getattr(ours.value, "line", None) == getattr(theirs.value, "line", None)


def test_low_rank_has_no_qps_form():
    with pytest.raises(ValueError):
        aqio.write_qps(instances.build("rqp:20:12:low_rank:0.3:5"))


QPS_FIXTURE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "qps_mixed_400.qps")


def test_qps_fixture_is_the_generator_output():
    """tests/golden/qps_mixed_400.qps is exactly oracle/gen_qps_fixture.py's output."""
    import gen_qps_fixture

    with open(QPS_FIXTURE) as f:
        assert f.read() == gen_qps_fixture.build()


@needs_ref
def test_qps_fixture_parses_like_reference():
    """The real-instance parity file (every reader convention): our reader and
    the reference's give the same problem, bit for bit."""
    from anchorqp import qps as rq

    text = open(QPS_FIXTURE).read()
    ours, theirs = aqio.parse_qps(text), rq.parse_qps(text)
    assert ours.objective_constant == theirs.objective_constant == 12.5
    same_problem(ours.problem, theirs.problem)
    p = ours.problem
    lo, hi = p.con_bounds.lower, p.con_bounds.upper
    assert np.sum(np.isfinite(lo) & np.isfinite(hi) & (lo < hi)) >= 30  # ranged rows
    assert np.sum(~np.isfinite(lo) & ~np.isfinite(hi)) == 2             # the two free N rows
    vlo, vhi = p.var_bounds.lower, p.var_bounds.upper
    assert np.any(~np.isfinite(vlo) & np.isfinite(vhi) & (vhi < 0))     # negative UP dropped the lower bound
    assert np.any(vlo == vhi)                                           # FX
