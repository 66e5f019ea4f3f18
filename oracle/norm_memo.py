"""TEST INFRASTRUCTURE ONLY: recorded results of the reference's own
``estimate_norm`` (aq/linalg.py:287-312) on the big bench instances.

On C5 (A: 5e7 x 5e7, 5e8 nonzeros) the reference's power iteration (100 x
A'A on one core) takes ~6 min of a reference-arm run whose timed region is
outer iterations [W, W+K) only -- initialisation is outside it.  To keep the
arm within its time limit, ``patch(aq)`` wraps ``anchorqp.engine
.estimate_norm`` so that for a matrix whose fingerprint (shape, nnz, a strided
sample of indptr/indices/data) and (iters, seed) match a recording it returns
the recorded float -- the value the very same reference function returned on
the very same matrix when it was recorded here with

    python oracle/norm_memo.py record c5:5e7:5000:0

Any other matrix falls through to the unmodified function.  The recorded
value is bitwise what the reference computes, so the trajectory is unchanged
(tests/test_oracle.py re-derives a small recording end to end).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
MEMO = os.path.join(ROOT, "tests", "golden", "ref_norm_memo.json")


def fingerprint(a) -> str:
    """Cheap identity of a CSR: shape, nnz and ~4096 strided samples of each array."""
    import numpy as np

    h = hashlib.sha256()
    h.update(f"{a.rows}:{a.cols}:{a.nnz}".encode())
    for arr in (np.asarray(a.indptr), np.asarray(a.indices), np.asarray(a.data)):
        step = max(1, arr.size // 4096)
        h.update(np.ascontiguousarray(arr[::step]).tobytes())
        if arr.size:
            h.update(np.ascontiguousarray(arr[-1:]).tobytes())
    return h.hexdigest()


def _load():
    try:
        with open(MEMO) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def patch(aq):
    """Route ``anchorqp.engine.estimate_norm`` through the recordings."""
    import anchorqp.engine as eng

    orig = getattr(eng.estimate_norm, "__wrapped__", eng.estimate_norm)
    memo = _load()

    def estimate_norm(a, iters=100, seed=0):
        rec = memo.get(fingerprint(a))
        if rec is not None and rec["iters"] == iters and rec["seed"] == seed:
            return float.fromhex(rec["value_hex"])
        return orig(a, iters, seed)

    estimate_norm.__wrapped__ = orig
    eng.estimate_norm = estimate_norm
    return estimate_norm


def record(spec: str, iters: int = 100, seed: int = 0):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    import instances
    import refbridge

    aq = refbridge.load_reference()
    assert aq is not None and aq.active_backend() == "cython"
    import anchorqp.linalg as L

    prob = refbridge.to_reference(instances.build(spec), aq)
    t0 = time.time()
    val = L.estimate_norm(prob.constraint_matrix, iters, seed)
    secs = time.time() - t0
    memo = _load()
    memo[fingerprint(prob.constraint_matrix)] = dict(spec=spec, iters=iters, seed=seed, value=val,
                                                     value_hex=float(val).hex(), seconds=secs)
    with open(MEMO, "w") as f:
        json.dump(memo, f, indent=1, sort_keys=True)
    print(json.dumps(dict(spec=spec, value=val, seconds=secs)))


if __name__ == "__main__":
    if len(sys.argv) >= 3 and sys.argv[1] == "record":
        record(sys.argv[2])
    else:
        print(__doc__)
