"""LP data model of the drop-in: the types the batched-solve path consumes and returns.

Restates the hot-path subset of the reference data model
(/root/reference/pkg/src/batchlp/model.py): ``Status`` (model.py:29-33),
``StandardFormLP`` (:97-115), ``standard_form`` (:118-123), ``SolveOutcome``
(:126-141) and ``validate`` (:263-301), with the same field names, string
values and violation messages so callers and tests written against the
reference work unchanged.  General-form lowering (GeneralLP, standardize,
VariableMap) and the MPS reader are host-side ingest in general.py / mps.py
(SURVEY.md §8(f) row 2).

The batch path does not call ``validate`` per LP: the kernels flag non-finite
inputs while building the tableau (BLP_STATUS_INVALID) and ``validate`` is
called only on the first flagged LP, to reproduce the reference's message.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np


class Status(Enum):
    OPTIMAL = "optimal"
    UNBOUNDED = "unbounded"
    INFEASIBLE = "infeasible"
    ITERATION_LIMIT = "iteration_limit"


# BLP_STATUS_* code -> Status (include/blp.h)
STATUS_BY_CODE = (Status.OPTIMAL, Status.UNBOUNDED, Status.INFEASIBLE, Status.ITERATION_LIMIT)


@dataclass(frozen=True)
class StandardFormLP:
    """maximize c.x  s.t.  A.x <= b,  x >= 0  (fp64; arrays treated as immutable)."""

    c: np.ndarray   # (n,)
    A: np.ndarray   # (m, n)
    b: np.ndarray   # (m,)

    @property
    def n(self) -> int:
        return len(self.c)

    @property
    def m(self) -> int:
        return len(self.b)


def standard_form(c, A, b) -> StandardFormLP:
    """Coerce sequences into a float64 StandardFormLP (model.py:118-123)."""
    c = np.asarray(c, dtype=float)
    b = np.asarray(b, dtype=float)
    A = np.asarray(A, dtype=float).reshape(len(b), len(c))
    return StandardFormLP(c=c, A=A, b=b)


@dataclass(frozen=True)
class SolveOutcome:
    """Terminal state of one solve; objective/point present iff OPTIMAL."""

    status: Status
    objective_value: float | None = None
    primal_point: np.ndarray | None = None
    iterations_phase1: int = 0
    iterations_phase2: int = 0

    def is_optimal(self) -> bool:
        return self.status is Status.OPTIMAL


def validate(lp: StandardFormLP) -> list[str]:
    """Violation strings for one LP; empty means valid (model.py:263-301)."""
    out: list[str] = []
    try:
        n = len(lp.c)
    except TypeError:
        return ["c is not a vector"]
    cvec = np.asarray(lp.c, dtype=float)
    out.extend(f"c[{j}] is not finite" for j in np.flatnonzero(~np.isfinite(cvec)))
    rows = list(lp.A)
    try:
        m = len(lp.b)
    except TypeError:
        return out + ["b is not a vector"]
    if len(rows) != m:
        out.append(f"A has {len(rows)} rows, expected {m}")
    for i, row in enumerate(rows):
        try:
            vals = np.atleast_1d(np.asarray(row, dtype=float))
        except (TypeError, ValueError):
            out.append(f"row {i} is not numeric")
            continue
        if len(vals) != n:
            out.append(f"row {i} has {len(vals)} coefficients, expected {n}")
            continue
        out.extend(f"A[{i}][{j}] is not finite" for j in np.flatnonzero(~np.isfinite(vals)))
    bvec = np.asarray(lp.b, dtype=float)
    out.extend(f"b[{i}] is not finite" for i in np.flatnonzero(~np.isfinite(bvec)))
    return out


def invalid_message(violations: list[str]) -> str:
    """The ValueError text solve() raises (simplex.py:162-164)."""
    return "invalid LP: " + "; ".join(violations)
