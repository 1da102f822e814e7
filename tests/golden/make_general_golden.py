"""Golden fixtures for general-form ingest, made by running the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_general_golden.py

Writes
  mps.json      MPS texts (the reference's fixture files, hand-written edge
                cases and seeded token-soup fuzz) with the reference parser's
                model or ParseError, its warnings, the lowered GeneralLP (or
                UnsupportedFeature), the standardized LP + VariableMap and
                the recovered outcome of the reference's own solve.
  general.json  seeded general LPs (mixed senses / relations / bounds, the
                shape family of the reference's test_model.py strategy) with
                the same standardize / solve / recover records.
Floats are written with repr (JSON NaN / Infinity tokens allowed).
"""
from __future__ import annotations

import json
import sys
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import batchlp  # noqa: E402  (the reference)
from batchlp import (GeneralLP, InfeasibleBounds, ParseError, UnsupportedFeature,  # noqa: E402
                     lower_to_general, parse_mps, solve, standardize)

FIXTURES = Path("/root/reference/pkg/fixtures")
CODES = {"optimal": 0, "unbounded": 1, "infeasible": 2, "iteration_limit": 3}


def floats(a) -> list:
    return [float(v) for v in np.asarray(a, dtype=float).ravel()]


def model_record(m) -> dict:
    return dict(name=m.name, sense=m.objective_sense.value, objective_row=m.objective_row,
                row_types=m.row_types, row_order=m.row_order, column_order=m.column_order,
                entries=[[k[0], k[1], float(v)] for k, v in m.entries.items()],
                rhs=[[k, float(v)] for k, v in m.rhs.items()],
                ranges=[[k, float(v)] for k, v in m.ranges.items()],
                bounds=[[t, v, None if x is None else float(x)] for t, v, x in m.bounds],
                integral=sorted(m.integral_columns))


def general_record(g) -> dict:
    return dict(sense=g.sense.value, c=floats(g.c), rows=floats(g.rows), k=int(g.num_rows), n=int(g.num_vars),
                relations=[r.value for r in g.relations], rhs=floats(g.rhs), lower=floats(g.lower),
                upper=floats(g.upper), row_names=list(g.row_names), col_names=list(g.col_names))


def lowered_record(g) -> dict:
    """standardize + the reference's solve + recover_outcome."""
    try:
        lp, vm = standardize(g)
    except InfeasibleBounds as err:
        return dict(error="InfeasibleBounds", message=str(err))
    out = solve(lp)
    rec = vm.recover_outcome(out)
    return dict(m=int(lp.m), n=int(lp.n), A=floats(lp.A), b=floats(lp.b), c=floats(lp.c),
                vmap=dict(sense=vm.sense.value, offset=float(vm.offset), shift=floats(vm.shift),
                          plus_col=[int(v) for v in vm.plus_col], minus_col=[int(v) for v in vm.minus_col],
                          num_standard_vars=int(vm.num_standard_vars)),
                std=dict(status=CODES[out.status.value], it1=out.iterations_phase1, it2=out.iterations_phase2,
                         objective=None if out.objective_value is None else float(out.objective_value),
                         x=None if out.primal_point is None else floats(out.primal_point)),
                outcome=dict(status=CODES[rec.status.value],
                             objective=None if rec.objective_value is None else float(rec.objective_value),
                             x=None if rec.primal_point is None else floats(rec.primal_point)))


def mps_record(name: str, text: str) -> dict:
    rec = dict(name=name, text=text)
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        try:
            model = parse_mps(text)
        except ParseError as err:
            rec.update(parse_error=str(err), line_no=err.line_no)
            model = None
        rec["parse_warnings"] = [str(w.message) for w in caught]
    if model is None:
        return rec
    rec["model"] = model_record(model)
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        try:
            g = lower_to_general(model)
        except UnsupportedFeature as err:
            rec.update(lower_error=str(err))
            g = None
        rec["lower_warnings"] = [str(w.message) for w in caught]
    if g is not None:
        rec["general"] = general_record(g)
        rec["lowered"] = lowered_record(g)
    return rec


# Hand-written edge cases covering each reader rule (mps.py:79-311).
BASE = """NAME          EDGE
ROWS
 N  cost
 L  lim1
 G  lim2
COLUMNS
    x1        cost      2.0        lim1      1.0
    x1        lim2      1.0
    x2        cost      -3.0       lim1      2.0
RHS
    rhs       lim1      8.0        lim2      1.0
ENDATA
"""
EDGE = {
    "base": BASE,
    "objsense_max_header": BASE.replace("NAME          EDGE\n", "NAME          EDGE\nOBJSENSE MAX\n"),
    "objsense_section": "OBJSENSE\n    MAXIMIZE\n" + BASE,
    "objsense_bad": "OBJSENSE\n    SIDEWAYS\n" + BASE,
    "no_endata": BASE.replace("ENDATA\n", ""),
    "empty": "",
    "comments_only": "* nothing here\n\n   \n",
    "unknown_section": "FOO\n" + BASE,
    "data_outside": "   x1 cost 1.0\n" + BASE,
    "name_then_data": "NAME X\n  stray tokens\n" + BASE,
    "rows_short": BASE.replace(" L  lim1", " L"),
    "rows_bad_type": BASE.replace(" G  lim2", " Q  lim2"),
    "rows_duplicate": BASE.replace(" G  lim2", " G  lim1"),
    "extra_n_row": BASE.replace(" L  lim1", " N  spare\n L  lim1").replace(
        "    x2        cost      -3.0       lim1      2.0", "    x2        cost      -3.0       spare     7.0"),
    "no_objective": BASE.replace(" N  cost\n", "").replace("cost      2.0        ", "").replace(
        "    x2        cost      -3.0       lim1      2.0", "    x2        lim1      2.0"),
    "columns_odd": BASE.replace("    x1        lim2      1.0", "    x1        lim2"),
    "columns_undeclared": BASE.replace("x1        lim2      1.0", "x1        lim9      1.0"),
    "columns_bad_number": BASE.replace("-3.0", "-3.0.0"),
    "columns_inf": BASE.replace("-3.0", "1e999"),
    "columns_nan": BASE.replace("-3.0", "nan"),
    "columns_duplicate": BASE.replace("    x1        lim2      1.0",
                                      "    x1        lim2      1.0\n    x1        lim1      0.5"),
    "marker_int": BASE.replace("COLUMNS\n", "COLUMNS\n    M1        'MARKER'                 'INTORG'\n").replace(
        "    x2 ", "    M2        'MARKER'                 'INTEND'\n    x2 "),
    "marker_bad": BASE.replace("COLUMNS\n", "COLUMNS\n    M1        'MARKER'                 'WHAT'\n"),
    "rhs_objective": BASE.replace("lim2      1.0\nENDATA", "lim2      1.0        cost      4.0\nENDATA"),
    "rhs_undeclared": BASE.replace("lim2      1.0\nENDATA", "lim7      1.0\nENDATA"),
    "rhs_duplicate": BASE.replace("ENDATA", "    rhs       lim1      9.0\nENDATA"),
    "rhs_no_setname": BASE.replace("    rhs       lim1      8.0        lim2      1.0", "    lim1 8.0 lim2 1.0"),
    "rows_without_rhs": BASE.replace("RHS\n    rhs       lim1      8.0        lim2      1.0\n", ""),
    "ranges_l": BASE.replace("ENDATA", "RANGES\n    rng       lim1      3.0\nENDATA"),
    "ranges_l_negative": BASE.replace("ENDATA", "RANGES\n    rng       lim1      -3.0\nENDATA"),
    "ranges_g": BASE.replace("ENDATA", "RANGES\n    rng       lim2      2.5\nENDATA"),
    "ranges_e_pos": BASE.replace(" G  lim2", " E  lim2").replace("ENDATA", "RANGES\n    rng   lim2   2.0\nENDATA"),
    "ranges_e_neg": BASE.replace(" G  lim2", " E  lim2").replace("ENDATA", "RANGES\n    rng   lim2   -2.0\nENDATA"),
    "ranges_objective": BASE.replace("ENDATA", "RANGES\n    rng       cost      1.0\nENDATA"),
    "ranges_undeclared": BASE.replace("ENDATA", "RANGES\n    rng       nope      1.0\nENDATA"),
    "bounds_all": BASE.replace("ENDATA", "BOUNDS\n UP BND x1 4.0\n LO BND x2 -1.0\n FX BND x2 0.5\n"
                                          " PL BND x1\nENDATA"),
    "bounds_no_setname": BASE.replace("ENDATA", "BOUNDS\n UP x1 4.0\n MI x2\nENDATA"),
    "bounds_fr": BASE.replace("ENDATA", "BOUNDS\n FR BND x2\nENDATA"),
    "bounds_mi_up": BASE.replace("ENDATA", "BOUNDS\n MI BND x1\n UP BND x1 3.0\nENDATA"),
    "bounds_negative_up": BASE.replace("ENDATA", "BOUNDS\n UP BND x1 -2.0\nENDATA"),
    "bounds_short": BASE.replace("ENDATA", "BOUNDS\n UP\nENDATA"),
    "bounds_bad_type": BASE.replace("ENDATA", "BOUNDS\n XX BND x1 1.0\nENDATA"),
    "bounds_no_value": BASE.replace("ENDATA", "BOUNDS\n UP BND\nENDATA"),
    "bounds_undeclared": BASE.replace("ENDATA", "BOUNDS\n UP BND zz 1.0\nENDATA"),
    "bounds_bv": BASE.replace("ENDATA", "BOUNDS\n BV BND x1\nENDATA"),
    "bounds_ui": BASE.replace("ENDATA", "BOUNDS\n UI BND x2 3.0\nENDATA"),
    "bounds_infeasible": BASE.replace("ENDATA", "BOUNDS\n LO BND x1 5.0\n UP BND x1 2.0\nENDATA"),
    "free_format_flush_left": "NAME FREE\nROWS\nN obj\nL c1\nCOLUMNS\nx obj 1 c1 1\ny obj 2 c1 1\nRHS\n"
                              "rhs c1 5\nENDATA\n",
    "free_format_keyword_name": "NAME KW\nROWS\n N obj\n L c1\nCOLUMNS\nRHS obj 1 c1 1\nRHS\n rhs c1 3\nENDATA\n",
    "lowercase_keywords": BASE.replace("ROWS", "rows").replace("COLUMNS", "columns"),
    "tabs_and_cr": BASE.replace("    ", "\t").replace("\n", "\r\n"),
    "after_endata": BASE + "GARBAGE after the end\n",
    "unbounded_min": "NAME U\nROWS\n N obj\n G c1\nCOLUMNS\n x obj -1.0 c1 1.0\nRHS\n rhs c1 1.0\nENDATA\n",
    "infeasible_pair": "NAME I\nROWS\n N obj\n L c1\n G c2\nCOLUMNS\n x obj 1.0 c1 1.0\n x c2 1.0\n"
                       "RHS\n rhs c1 1.0 c2 3.0\nENDATA\n",
    "equality_free": "NAME E\nROWS\n N obj\n E bal\n L cap\nCOLUMNS\n x obj 2 bal 1\n x cap 1\n y obj 1 bal 1\n"
                     "RHS\n rhs bal 4 cap 3\nBOUNDS\n FR b y\nENDATA\n",
}

VOCAB = ["NAME", "ROWS", "COLUMNS", "RHS", "RANGES", "BOUNDS", "ENDATA", "OBJSENSE", "MAX", "MIN", "N", "L",
         "G", "E", "UP", "LO", "FX", "FR", "MI", "PL", "BV", "obj", "c1", "c2", "x", "y", "rhs", "1.0", "-2",
         "3e2", "nan", "inf", "'MARKER'", "'INTORG'", "'INTEND'", "*", "1e999", "0", "abc"]


def fuzz_texts(count: int, seed: int) -> list[str]:
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        lines = []
        for _ in range(int(rng.integers(1, 14))):
            toks = [VOCAB[int(i)] for i in rng.integers(0, len(VOCAB), int(rng.integers(1, 6)))]
            lines.append((" " if rng.random() < 0.5 else "") + " ".join(toks))
        if rng.random() < 0.6:
            lines.append("ENDATA")
        out.append("\n".join(lines) + "\n")
    # grammatical skeletons with one random defect each
    for k in range(count):
        t = BASE.splitlines()
        i = int(rng.integers(0, len(t)))
        t[i] = " ".join(VOCAB[int(j)] for j in rng.integers(0, len(VOCAB), int(rng.integers(0, 5))))
        out.append("\n".join(t) + "\n")
    return out


def general_lps(count: int, seed: int):
    """Seeded family shaped like test_model.py's general_lps strategy (:111-135)."""
    rng = np.random.default_rng(seed)
    for _ in range(count):
        n, k = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        rows = rng.integers(-6, 7, size=(k, n)).astype(float)
        rhs = rng.integers(-8, 9, size=k).astype(float)
        rels = [["<=", ">=", "="][int(i)] for i in rng.integers(0, 3, size=k)]
        c = rng.integers(-6, 7, size=n).astype(float)
        lower, upper = np.zeros(n), np.full(n, np.inf)
        for j in range(n):
            kind = int(rng.integers(0, 4))
            if kind == 1:
                lower[j] = rng.integers(-4, 3)
                upper[j] = lower[j] + rng.integers(0, 7)
            elif kind == 2:
                lower[j] = -np.inf
                upper[j] = rng.integers(-2, 7)
            elif kind == 3:
                lower[j] = rng.integers(-4, 1)
        yield GeneralLP.build(["min", "max"][int(rng.integers(0, 2))], c, rows, rels, rhs, lower, upper)


def main():
    recs = [mps_record(f"fixture:{p.name}", p.read_text()) for p in sorted(FIXTURES.glob("*.mps"))]
    recs += [mps_record(f"edge:{k}", v) for k, v in EDGE.items()]
    recs += [mps_record(f"fuzz:{i}", t) for i, t in enumerate(fuzz_texts(150, 8557))]
    (HERE / "mps.json").write_text(json.dumps(dict(reference=f"batchlp {batchlp.__version__}", records=recs)))
    gens = []
    for i, g in enumerate(general_lps(400, 1802)):
        gens.append(dict(name=f"general:{i}", general=general_record(g), lowered=lowered_record(g)))
    # fixed-layout family for the packed batch path: same relations / bounds pattern, varied data
    rng = np.random.default_rng(855)
    for i in range(300):
        rows = rng.integers(-5, 6, size=(4, 3)).astype(float)
        g = GeneralLP.build(["min", "max"][i % 2], rng.integers(-5, 6, size=3).astype(float), rows,
                            ["<=", ">=", "=", "<="], rng.integers(-6, 10, size=4).astype(float),
                            lower=[-np.inf, float(rng.integers(-3, 1)), 0.0],
                            upper=[float(rng.integers(0, 6)), np.inf, float(rng.integers(1, 8))])
        gens.append(dict(name=f"family:{i}", general=general_record(g), lowered=lowered_record(g)))
    (HERE / "general.json").write_text(json.dumps(dict(reference=f"batchlp {batchlp.__version__}",
                                                       records=gens)))
    print(len(recs), "mps records;", len(gens), "general records")


if __name__ == "__main__":
    main()
