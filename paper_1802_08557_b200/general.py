"""General-form ingest for the batched path.

A ``GeneralLP`` (min/max sense, <=/>=/= rows, variable bounds) is lowered to
the maximisation standard form the kernels solve, and a ``VariableMap``
undoes the lowering on the solver's outputs.  Semantics follow the reference
(/root/reference/pkg/src/batchlp/model.py): ``Sense``/``Relation`` (:19-26),
``InfeasibleBounds`` (:36-37), ``GeneralLP`` (:40-94), ``VariableMap``
(:144-181) and ``standardize`` (:184-260), with the same rounding: every
lowered coefficient is a copy or a negation, and the two dot products the
reference forms (``row @ shift`` per row, ``c @ shift``) are taken with the
same 1-D numpy call so the lowered LPs are bitwise the reference's.

The batch layer is new: ``standardize_batch`` lowers many general LPs into
one packed (A, b, c) batch for ``batch_solve_arrays``, and ``recover_batch``
maps the packed GPU outputs back with one gather per variable-map layout.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np

from .model import SolveOutcome, StandardFormLP, Status


class Sense(Enum):
    MIN = "min"
    MAX = "max"


class Relation(Enum):
    LE = "<="
    GE = ">="
    EQ = "="


class InfeasibleBounds(Exception):
    """A variable's lower bound exceeds its upper bound."""


@dataclass(frozen=True)
class GeneralLP:
    """sense c.x  s.t.  rows[i].x (<=|>=|=) rhs[i],  lower <= x <= upper  (model.py:40-94).

    Arrays are treated as immutable after construction.
    """

    sense: Sense
    c: np.ndarray                      # (n,)
    rows: np.ndarray                   # (k, n)
    relations: tuple[Relation, ...]    # (k,)
    rhs: np.ndarray                    # (k,)
    lower: np.ndarray                  # (n,), -inf allowed
    upper: np.ndarray                  # (n,), +inf allowed
    row_names: tuple[str, ...] = ()
    col_names: tuple[str, ...] = ()

    def __post_init__(self):
        n, k = self.c.shape[0], self.rhs.shape[0]
        if self.rows.shape != (k, n):
            raise ValueError(f"rows has shape {self.rows.shape}, expected ({k}, {n})")
        if len(self.relations) != k:
            raise ValueError(f"{len(self.relations)} relations for {k} rows")
        if self.lower.shape != (n,) or self.upper.shape != (n,):
            raise ValueError("bounds must both have length n")
        if not self.row_names:
            object.__setattr__(self, "row_names", tuple(f"r{i}" for i in range(k)))
        if not self.col_names:
            object.__setattr__(self, "col_names", tuple(f"x{j}" for j in range(n)))
        if len(set(self.row_names)) != k or len(set(self.col_names)) != n:
            raise ValueError("row/column names must be unique")

    @property
    def num_vars(self) -> int:
        return self.c.shape[0]

    @property
    def num_rows(self) -> int:
        return self.rhs.shape[0]

    @classmethod
    def build(cls, sense, c, rows, relations, rhs, lower=None, upper=None,
              row_names=(), col_names=()) -> "GeneralLP":
        """From plain sequences; bounds default to [0, +inf) (model.py:80-94)."""
        c = np.asarray(c, dtype=float)
        n = c.shape[0]
        return cls(sense if isinstance(sense, Sense) else Sense(sense),
                   c,
                   np.asarray(rows, dtype=float).reshape(-1, n),
                   tuple(r if isinstance(r, Relation) else Relation(r) for r in relations),
                   np.asarray(rhs, dtype=float),
                   np.zeros(n) if lower is None else np.asarray(lower, dtype=float),
                   np.full(n, np.inf) if upper is None else np.asarray(upper, dtype=float),
                   tuple(row_names), tuple(col_names))


@dataclass(frozen=True)
class VariableMap:
    """Undo record of ``standardize`` (model.py:144-181).

    Original variable j is standard column ``plus_col[j]`` minus, when it was
    split because it is unbounded below, column ``minus_col[j]`` (-1 if not),
    plus the lower-bound ``shift[j]``; ``offset`` = c.shift.
    """

    sense: Sense
    offset: float
    shift: np.ndarray
    plus_col: np.ndarray
    minus_col: np.ndarray
    num_standard_vars: int

    def recover_point(self, x_std: np.ndarray) -> np.ndarray:
        x = np.array(x_std[self.plus_col], dtype=float)
        split = self.minus_col >= 0
        x[split] -= x_std[self.minus_col[split]]
        return x + self.shift

    def recover_objective(self, standard_value: float) -> float:
        return (1.0 if self.sense is Sense.MAX else -1.0) * standard_value + self.offset

    def recover_outcome(self, outcome: SolveOutcome) -> SolveOutcome:
        if not outcome.is_optimal():
            return outcome
        return SolveOutcome(status=outcome.status,
                            objective_value=self.recover_objective(outcome.objective_value),
                            primal_point=self.recover_point(outcome.primal_point),
                            iterations_phase1=outcome.iterations_phase1,
                            iterations_phase2=outcome.iterations_phase2)

    def layout_key(self) -> tuple:
        """Maps with equal keys recover with the same gather (recover_batch)."""
        return (self.num_standard_vars, self.plus_col.tobytes(), self.minus_col.tobytes())


def _column_layout(lower: np.ndarray):
    """Standard columns of each variable: one, or a +/- pair when unbounded below."""
    split = ~np.isfinite(lower)
    width = 1 + split.astype(np.int64)
    plus = np.cumsum(width) - width
    minus = np.where(split, plus + 1, -1)
    shift = np.where(split, 0.0, lower)
    return plus.astype(int), minus.astype(int), shift, int(width.sum())


def _widen(block: np.ndarray, plus: np.ndarray, minus: np.ndarray, n_std: int) -> np.ndarray:
    """Rows over the original variables -> rows over the standard columns."""
    out = np.zeros(block.shape[:-1] + (n_std,))
    out[..., plus] = block
    split = minus >= 0
    out[..., minus[split]] = -block[..., split]
    return out


def standardize(glp: GeneralLP) -> tuple[StandardFormLP, VariableMap]:
    """Lower to max c.x, A x <= b, x >= 0 (model.py:184-260).

    Row order: for each general row, its <= form unless it is >=, then its
    negated form unless it is <=; then one row per finite upper bound in
    variable order.  MIN negates the objective.
    """
    lower, upper = glp.lower, glp.upper
    bad = np.flatnonzero(lower > upper)
    if bad.size:
        j = int(bad[0])
        raise InfeasibleBounds(f"variable {glp.col_names[j]!r}: lower {lower[j]} > upper {upper[j]}")
    plus, minus, shift, n_std = _column_layout(lower)

    src, sign = [], []
    for i, rel in enumerate(glp.relations):
        if rel is not Relation.GE:
            src.append(i)
            sign.append(1.0)
        if rel is not Relation.LE:
            src.append(i)
            sign.append(-1.0)
    src = np.asarray(src, dtype=int)
    sign = np.asarray(sign)
    wide = _widen(glp.rows, plus, minus, n_std)
    # rhs - row.shift, the dot per row as the reference forms it (1-D numpy dot)
    shifted = np.array([glp.rhs[i] - float(glp.rows[i] @ shift) for i in range(glp.num_rows)])
    blocks = [np.where(sign[:, None] > 0, wide[src], -wide[src]) if src.size else np.zeros((0, n_std))]
    rhs = [np.where(sign > 0, shifted[src], -shifted[src]) if src.size else np.zeros(0)]

    capped = np.flatnonzero(np.isfinite(upper))
    if capped.size:
        cap = np.zeros((capped.size, n_std))
        cap[np.arange(capped.size), plus[capped]] = 1.0
        has_minus = minus[capped] >= 0
        cap[np.flatnonzero(has_minus), minus[capped][has_minus]] = -1.0
        blocks.append(cap)
        rhs.append(upper[capped] - shift[capped])

    c_std = _widen(glp.c, plus, minus, n_std)
    if glp.sense is Sense.MIN:
        c_std = -c_std
    A = np.vstack(blocks)
    b = np.concatenate(rhs).astype(float)
    lp = StandardFormLP(c=c_std, A=A if A.shape[0] else np.zeros((0, n_std)), b=b)
    return lp, VariableMap(sense=glp.sense, offset=float(glp.c @ shift), shift=shift,
                           plus_col=plus, minus_col=minus, num_standard_vars=n_std)


# ---------------------------------------------------------------- batch layer

def standardize_batch(glps: Sequence[GeneralLP]):
    """Lower many general LPs into one packed batch: (A [B,m,n], b [B,m], c [B,n], maps).

    Every LP must lower to the same (m, n) (the kernels batch one shape).
    """
    lps, maps = [], []
    for g in glps:
        lp, vm = standardize(g)
        lps.append(lp)
        maps.append(vm)
    if not lps:
        return np.zeros((0, 0, 0)), np.zeros((0, 0)), np.zeros((0, 0)), maps
    m, n = lps[0].m, lps[0].n
    for k, lp in enumerate(lps):
        if (lp.m, lp.n) != (m, n):
            raise ValueError(f"general LP {k} lowers to ({lp.m}, {lp.n}), batch shape is ({m}, {n})")
    A = np.stack([lp.A for lp in lps]).reshape(len(lps), m, n)
    b = np.stack([lp.b for lp in lps]).reshape(len(lps), m)
    c = np.stack([lp.c for lp in lps]).reshape(len(lps), n)
    return A, b, c, maps


@dataclass
class GeneralBatch:
    """Recovered outputs of a general-form batch: objective NaN and x zero unless optimal."""

    status: np.ndarray         # int8 [B], BLP status codes
    objective: np.ndarray      # f64 [B]
    x: list                    # per-LP original-variable points (lengths may differ)
    iterations_phase1: np.ndarray
    iterations_phase2: np.ndarray

    def outcome(self, k: int) -> SolveOutcome:
        from .model import STATUS_BY_CODE
        st = STATUS_BY_CODE[int(self.status[k])]
        opt = st is Status.OPTIMAL
        return SolveOutcome(status=st, objective_value=float(self.objective[k]) if opt else None,
                            primal_point=self.x[k] if opt else None,
                            iterations_phase1=int(self.iterations_phase1[k]),
                            iterations_phase2=int(self.iterations_phase2[k]))


def recover_batch(maps: Sequence[VariableMap], result) -> GeneralBatch:
    """Apply each LP's VariableMap to packed solver outputs (a BatchArrays).

    LPs whose maps share a column layout are recovered with one gather over
    the whole group; arithmetic is the same elementwise ops as recover_point /
    recover_objective, so each row equals the per-LP recovery bitwise.
    """
    B = len(maps)
    status = np.asarray(result.status)
    opt = status == 0
    objective = np.full(B, np.nan)
    xs: list = [None] * B
    groups: dict = {}
    for k, vm in enumerate(maps):
        groups.setdefault(vm.layout_key(), []).append(k)
    X = np.asarray(result.x)
    for idx in groups.values():
        vm0 = maps[idx[0]]
        idx = np.asarray(idx)
        split = vm0.minus_col >= 0
        pts = np.array(X[idx][:, vm0.plus_col], dtype=float)
        pts[:, split] -= X[idx][:, vm0.minus_col[split]]
        pts += np.stack([maps[k].shift for k in idx]).reshape(len(idx), -1)
        sgn = np.array([1.0 if maps[k].sense is Sense.MAX else -1.0 for k in idx])
        off = np.array([maps[k].offset for k in idx])
        obj = sgn * np.asarray(result.objective)[idx] + off
        for j, k in enumerate(idx):
            if opt[k]:
                objective[k] = obj[j]
                xs[k] = pts[j]
            else:
                xs[k] = np.zeros(pts.shape[1])
    return GeneralBatch(status=status, objective=objective, x=xs,
                        iterations_phase1=np.asarray(result.iterations_phase1),
                        iterations_phase2=np.asarray(result.iterations_phase2))


def solve_general(glp: GeneralLP, limits=None) -> SolveOutcome:
    """standardize -> GPU solve -> recover (one LP)."""
    from .simplex import SolverLimits, solve
    lp, vm = standardize(glp)
    return vm.recover_outcome(solve(lp, limits or SolverLimits()))


def batch_solve_general(glps: Sequence[GeneralLP], limits=None) -> GeneralBatch:
    """Lower a same-shape family of general LPs, solve it in one GPU batch, map it back."""
    from .batch import batch_solve_arrays
    from .simplex import SolverLimits
    A, b, c, maps = standardize_batch(glps)
    res = batch_solve_arrays(A, b, c, limits or SolverLimits())
    return recover_batch(maps, res)
