"""Inner-solve policy types (reference ``anchorqp/inner.py:24-48``).

The BB projected-gradient solve itself runs on the device inside the outer
iteration graph (``csrc/aqp_solver.cu``: OpGrad / OpStep under a CUDA-graph
WHILE node); what stays here is the host-visible tolerance rule, used by the
solve loop's bookkeeping and by the tests.
"""

from __future__ import annotations

import dataclasses

BB_STEP_MIN = 1e-10
BB_STEP_MAX = 1e10


@dataclasses.dataclass(frozen=True)
class InnerTolerance:
    """Monotone non-increasing inner tolerance with a floor (inner.py:28-38)."""

    current: float
    floor: float = 1e-9
    scale: float = 5e-4

    def __post_init__(self):
        if self.current <= 0:
            raise ValueError("tolerance must be positive")


def update_tolerance(tol: InnerTolerance, omega: float, tau: float, primal_move: float) -> InnerTolerance:
    """min(current, max(scale * omega * move / tau, floor)) (inner.py:41-48)."""
    cand = max(tol.scale * omega * primal_move / tau, tol.floor)
    return dataclasses.replace(tol, current=min(tol.current, cand))
