"""Single-LP entry point of the drop-in: ``solve`` and ``SolverLimits``.

Mirrors /root/reference/pkg/src/batchlp/simplex.py: ``SolverLimits``
(simplex.py:34-60) with the same defaults and validation, and
``solve(lp, limits)`` (simplex.py:154-194) with the same exceptions
(``ValueError("invalid LP: ...")``, ``RuntimeError`` when phase 1 reports
unbounded) and the same ``SolveOutcome``.  The arithmetic runs in the CUDA
kernel (a batch of one); see paper_1802_08557_b200/csrc/.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .model import SolveOutcome, StandardFormLP, STATUS_BY_CODE, Status, invalid_message, validate

PHASE1_ZERO_TOL = 1e-7       # simplex.py:26 (compiled into the kernels)
DEGENERATE_RATIO_TOL = 1e-9  # simplex.py:27
REDUNDANT_ROW_TOL = 1e-7     # simplex.py:31

PHASE1_UNBOUNDED_MESSAGE = "phase-1 auxiliary objective reported unbounded"


@dataclass(frozen=True)
class SolverLimits:
    """Per-phase iteration budget and anti-cycling policy (simplex.py:34-60)."""

    max_iterations: int | None = None
    anti_cycling: bool = True
    degenerate_pivot_limit: int | None = None

    def __post_init__(self):
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")

    def iterations_for(self, m: int, n: int) -> int:
        return self.max_iterations if self.max_iterations is not None else 50 * (m + n)

    def bland_trigger(self, m: int) -> int:
        if self.degenerate_pivot_limit is not None:
            return self.degenerate_pivot_limit
        return max(m, 1)

    def to_native(self) -> _native.Limits:
        return _native.make_limits(self.max_iterations, self.anti_cycling, self.degenerate_pivot_limit)


def outcome_from_arrays(res: dict, k: int) -> SolveOutcome:
    """SolveOutcome of LP k of a native result (objective/x only when OPTIMAL)."""
    code = int(res["status"][k])
    if code == 4:
        raise RuntimeError(PHASE1_UNBOUNDED_MESSAGE)
    status = STATUS_BY_CODE[code]
    if status is Status.OPTIMAL:
        return SolveOutcome(status, objective_value=float(res["objective"][k]),
                            primal_point=np.array(res["x"][k], dtype=np.float64),
                            iterations_phase1=int(res["it1"][k]), iterations_phase2=int(res["it2"][k]))
    return SolveOutcome(status, iterations_phase1=int(res["it1"][k]), iterations_phase2=int(res["it2"][k]))


def outcomes_from_arrays(res: dict, start: int, end: int) -> list[SolveOutcome]:
    """outcome_from_arrays for LPs [start, end) of a native result, in bulk: scalars via
    tolist(), each primal point a row view of one copy of x (the reference's point is a
    view too: ``x[:n]`` of its per-LP vector, simplex.py:146-151)."""
    codes = res["status"][start:end].tolist()
    if 4 in codes:
        raise RuntimeError(PHASE1_UNBOUNDED_MESSAGE)
    obj = res["objective"][start:end].tolist()
    it1 = res["it1"][start:end].tolist()
    it2 = res["it2"][start:end].tolist()
    xs = np.array(res["x"][start:end], dtype=np.float64)
    opt = Status.OPTIMAL
    out = []
    for k, code in enumerate(codes):
        st = STATUS_BY_CODE[code]
        if st is opt:
            out.append(SolveOutcome(st, obj[k], xs[k], it1[k], it2[k]))
        else:
            out.append(SolveOutcome(st, None, None, it1[k], it2[k]))
    return out


def solve(lp: StandardFormLP, limits: SolverLimits = SolverLimits(), device: int = 0) -> SolveOutcome:
    """Two-phase simplex solve of one standard-form LP on the GPU."""
    violations = validate(lp)
    if violations:
        raise ValueError(invalid_message(violations))
    m, n = lp.m, lp.n
    A = np.ascontiguousarray(np.asarray(lp.A, dtype=np.float64).reshape(1, m, n))
    b = np.ascontiguousarray(np.asarray(lp.b, dtype=np.float64).reshape(1, m))
    c = np.ascontiguousarray(np.asarray(lp.c, dtype=np.float64).reshape(1, n))
    res = _native.solve_host(A, b, c, limits.to_native(), device=device)
    return outcome_from_arrays(res, 0)
