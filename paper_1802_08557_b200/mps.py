"""MPS reader (fixed or free format) feeding the general-form ingest.

Behaviour follows the reference reader (/root/reference/pkg/src/batchlp/mps.py):
whitespace-delimited, section-ordered parsing (NAME, OBJSENSE, ROWS,
COLUMNS, RHS, RANGES, BOUNDS, ENDATA); ``parse_mps`` is total, returning an
``MpsModel`` or raising ``ParseError`` carrying the line number, with the
reference's messages and warnings (mps.py:79-250); ``lower_to_general``
builds a ``GeneralLP`` with the MPS default MIN sense and the published
RANGES conventions (mps.py:253-311).
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

from .general import GeneralLP, Relation, Sense

SECTIONS = frozenset({"NAME", "OBJSENSE", "ROWS", "COLUMNS", "RHS", "RANGES", "BOUNDS", "ENDATA"})
ROW_KINDS = {"N": None, "L": Relation.LE, "G": Relation.GE, "E": Relation.EQ}
BOUND_KINDS = frozenset({"UP", "LO", "FX", "FR", "MI", "PL", "BV", "UI", "LI"})
NO_VALUE_BOUNDS = frozenset({"FR", "MI", "PL", "BV"})
INTEGER_BOUNDS = ("BV", "UI", "LI")


class ParseError(Exception):
    def __init__(self, message: str, line_no: int):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class UnsupportedFeature(Exception):
    """Integer / binary features, which a dense LP reader rejects."""


@dataclass
class MpsModel:
    name: str = ""
    objective_sense: Sense = Sense.MIN
    objective_row: str | None = None
    row_types: dict[str, str] = field(default_factory=dict)     # constraint row -> L/G/E
    row_order: list[str] = field(default_factory=list)
    column_order: list[str] = field(default_factory=list)
    entries: dict[tuple[str, str], float] = field(default_factory=dict)   # (column, row) -> value
    rhs: dict[str, float] = field(default_factory=dict)
    ranges: dict[str, float] = field(default_factory=dict)
    bounds: list[tuple[str, str, float | None]] = field(default_factory=list)
    integral_columns: set[str] = field(default_factory=set)


class _Reader:
    """One pass over the lines; ``section`` selects the data-line handler."""

    def __init__(self):
        self.model = MpsModel()
        self.declared: dict[str, str] = {}     # every ROWS name (N rows included) -> type
        self.columns: set[str] = set()
        self.section: str | None = None
        self.in_integer_block = False
        self.line = 0

    # -- helpers
    def fail(self, message: str):
        raise ParseError(message, self.line)

    def number(self, token: str) -> float:
        try:
            v = float(token)
        except ValueError:
            self.fail(f"malformed numeric {token!r}")
        if not np.isfinite(v):
            self.fail(f"non-finite numeric {token!r}")
        return v

    def row_value_pairs(self, f: list[str], kind: str):
        # odd field count: the first token names the RHS/RANGES set
        for k in range(len(f) % 2, len(f), 2):
            if f[k] not in self.declared:
                self.fail(f"{kind} entry references undeclared row {f[k]!r}")
            yield f[k], self.number(f[k + 1])

    def sense(self, token: str) -> Sense:
        w = token.upper()
        if w in ("MAX", "MAXIMIZE"):
            return Sense.MAX
        if w in ("MIN", "MINIMIZE"):
            return Sense.MIN
        self.fail(f"unknown OBJSENSE {token!r}")

    # -- section handlers
    def on_OBJSENSE(self, f):
        self.model.objective_sense = self.sense(f[0])

    def on_ROWS(self, f):
        if len(f) < 2:
            self.fail("ROWS line needs a type and a name")
        kind, name = f[0].upper(), f[1]
        if kind not in ROW_KINDS:
            self.fail(f"unknown row type {f[0]!r}")
        if name in self.declared:
            self.fail(f"duplicate row name {name!r}")
        self.declared[name] = kind
        if kind != "N":
            self.model.row_types[name] = kind
            self.model.row_order.append(name)
        elif self.model.objective_row is None:
            self.model.objective_row = name
        else:
            warnings.warn(f"extra objective row {name!r} ignored")

    def on_COLUMNS(self, f):
        if len(f) >= 3 and f[1] == "'MARKER'":
            tag = f[2].strip("'").upper()
            if tag not in ("INTORG", "INTEND"):
                self.fail(f"unknown marker {f[2]!r}")
            self.in_integer_block = tag == "INTORG"
            return
        if len(f) < 3 or len(f) % 2 == 0:
            self.fail("COLUMNS line needs a column name and (row, value) pairs")
        col = f[0]
        if col not in self.columns:
            self.columns.add(col)
            self.model.column_order.append(col)
        if self.in_integer_block:
            self.model.integral_columns.add(col)
        entries = self.model.entries
        for k in range(1, len(f), 2):
            row = f[k]
            if row not in self.declared:
                self.fail(f"COLUMNS entry references undeclared row {row!r}")
            v = self.number(f[k + 1])
            if (col, row) in entries:
                warnings.warn(f"duplicate entry for ({col}, {row}); values summed")
                entries[(col, row)] += v
            else:
                entries[(col, row)] = v

    def on_RHS(self, f):
        for row, v in self.row_value_pairs(f, "RHS"):
            if row in self.model.rhs:
                warnings.warn(f"duplicate RHS for row {row!r}; keeping the last value")
            self.model.rhs[row] = v

    def on_RANGES(self, f):
        for row, v in self.row_value_pairs(f, "RANGES"):
            if self.declared[row] == "N":
                warnings.warn(f"RANGES entry on objective row {row!r} ignored")
            else:
                self.model.ranges[row] = v

    def on_BOUNDS(self, f):
        if len(f) < 2:
            self.fail("BOUNDS line too short")
        kind = f[0].upper()
        if kind not in BOUND_KINDS:
            self.fail(f"unknown bound type {f[0]!r}")
        rest = f[1:]
        value = None
        if kind in NO_VALUE_BOUNDS:        # optional bound-set name before the column
            var = rest[1] if len(rest) >= 2 and rest[1] in self.columns else rest[0]
        elif len(rest) >= 3:
            var, value = rest[1], self.number(rest[2])
        elif len(rest) == 2 and rest[0] in self.columns:
            var, value = rest[0], self.number(rest[1])
        else:
            self.fail("bound entry needs a variable and a value")
        if var not in self.columns:
            self.fail(f"BOUNDS entry references undeclared column {var!r}")
        self.model.bounds.append((kind, var, value))

    # -- driver
    def header(self, f) -> bool:
        """Section header: returns True at ENDATA."""
        key = f[0].upper()
        self.section = key
        if key == "ENDATA":
            return True
        if key == "NAME":
            self.model.name = f[1] if len(f) > 1 else ""
        elif key == "OBJSENSE" and len(f) > 1:
            self.model.objective_sense = self.sense(f[1])
            self.section = None
        return False

    def run(self, text: str) -> MpsModel:
        ended = False
        for self.line, raw in enumerate(text.splitlines(), start=1):
            line = raw.rstrip()
            body = line.lstrip()
            if not body or body.startswith("*"):
                continue
            f = line.split()
            flush_left = not line[0].isspace()
            # A header carries the keyword plus at most one name; a longer
            # flush-left line is free-format data whose first name looks like one.
            if flush_left and f[0].upper() in SECTIONS and (f[0].upper() in ("NAME", "OBJSENSE") or len(f) <= 2):
                if self.header(f):
                    ended = True
                    break
                continue
            if self.section in (None, "NAME"):
                self.fail(f"unknown section {f[0]!r}" if flush_left else "data line outside any section")
            getattr(self, "on_" + self.section)(f)
        self.line = max(self.line, 1)
        if not ended:
            self.fail("missing ENDATA")
        if self.model.objective_row is None:
            self.fail("no objective (type N) row declared")
        return self.model


def parse_mps(text: str) -> MpsModel:
    """Parse MPS text; any defect raises ParseError with its line number."""
    return _Reader().run(text)


def lower_to_general(model: MpsModel) -> GeneralLP:
    """GeneralLP of a parsed model: MIN by default, variables in [0, +inf) unless bounded.

    A ranged L/G/E row becomes ``row <= hi`` (its own name) then
    ``row >= lo`` (name + "__rng").  Integer markers and BV/UI/LI bounds raise
    UnsupportedFeature.
    """
    if model.integral_columns:
        raise UnsupportedFeature("integer columns not supported (e.g. "
                                 + ", ".join(sorted(model.integral_columns)[:3]) + ")")
    for kind, var, _ in model.bounds:
        if kind in INTEGER_BOUNDS:
            raise UnsupportedFeature(f"{kind} bound on {var!r} not supported")

    cols = {name: j for j, name in enumerate(model.column_order)}
    rows_at = {name: i for i, name in enumerate(model.row_order)}
    n = len(cols)
    c = np.zeros(n)
    dense = np.zeros((len(rows_at), n))
    for (col, row), v in model.entries.items():
        if row == model.objective_row:
            c[cols[col]] = v
        elif row in rows_at:
            dense[rows_at[row], cols[col]] = v
    if model.objective_row in model.rhs:
        warnings.warn("RHS entry on the objective row ignored")

    out_rows, rels, rhs, names = [], [], [], []
    for i, name in enumerate(model.row_order):
        kind = model.row_types[name]
        b = model.rhs.get(name, 0.0)
        if name not in model.ranges:
            out_rows.append(dense[i])
            rels.append(ROW_KINDS[kind])
            rhs.append(b)
            names.append(name)
            continue
        r = model.ranges[name]
        if kind == "L":
            lo, hi = b - abs(r), b
        elif kind == "G":
            lo, hi = b, b + abs(r)
        else:
            lo, hi = (b, b + r) if r >= 0 else (b + r, b)
        out_rows += [dense[i], dense[i].copy()]
        rels += [Relation.LE, Relation.GE]
        rhs += [hi, lo]
        names += [name, f"{name}__rng"]

    lower, upper = np.zeros(n), np.full(n, np.inf)
    for kind, var, v in model.bounds:
        j = cols[var]
        if kind == "UP":
            upper[j] = v
            if v < 0 and lower[j] == 0:
                warnings.warn(f"negative UP bound on {var!r} with default lower bound 0")
        elif kind == "LO":
            lower[j] = v
        elif kind == "FX":
            lower[j] = upper[j] = v
        elif kind == "FR":
            lower[j], upper[j] = -np.inf, np.inf
        elif kind == "MI":
            lower[j] = -np.inf
        elif kind == "PL":
            upper[j] = np.inf

    return GeneralLP(sense=model.objective_sense, c=c,
                     rows=np.vstack(out_rows) if out_rows else np.zeros((0, n)),
                     relations=tuple(rels), rhs=np.asarray(rhs, dtype=float),
                     lower=lower, upper=upper, row_names=tuple(names),
                     col_names=tuple(model.column_order))
