"""GPU: many-instance batching (batch.solve_many / run_benchmark), SURVEY.md
§8(f) item 4 -- concurrent solves on one B200 return exactly what the solves
return alone, and the reference's benchmark records / SGM10 come out."""

import numpy as np
import pytest

import instances
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import batch, io as aqio

pytestmark = pytest.mark.gpu


def test_solve_many_equals_sequential(cuda):
    probs = [aq.random_qp(300 + 20 * s, 150, "sparse" if s % 3 else "diagonal", density=0.05, seed=s)
             for s in range(9)]
    prm = aq.SolverParams(eps_tol=1e-8)
    seq = [aq.solve(p, prm) for p in probs]
    par = batch.solve_many(probs, prm, streams=4)
    for a, b in zip(seq, par):
        assert a.status == b.status
        assert (a.outer_iterations, a.inner_iterations, a.restarts) == (b.outer_iterations, b.inner_iterations,
                                                                         b.restarts)
        assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y)


def test_run_benchmark_records_from_files(cuda, tmp_path):
    specs = ["rqp:300:150:sparse:0.05:7", "rqp:500:300:diagonal:0.02:5", "c4i:1e3:1"]
    paths = []
    for k, spec in enumerate(specs):
        f = tmp_path / (f"i{k}." + ("aqpz", "json", "qps")[k])
        aqio.save_problem(instances.build(spec), f)
        paths.append(f)
    bad = tmp_path / "zz_bad.qps"
    bad.write_text("NAME X\nFOO\n")
    recs = batch.run_benchmark(paths + [bad], aq.SolverParams(eps_tol=1e-8), streams=3)
    assert [r.instance for r in recs] == sorted(r.instance for r in recs)
    by = {r.instance: r for r in recs}
    assert by["i0.aqpz"].status == "optimal" and by["i1.json"].status == "optimal"
    assert by["i2.qps"].status == "primal_infeasible"
    assert by["zz_bad.qps"].status.startswith("error:")
    s = batch.summarize(recs, time_limit=60.0)
    assert s["instances"] == 4 and s["solved"] == 2 and s["failed"] == 2
    assert s["sgm10_seconds"] > 0.0
