"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package read-only
(sys.path += /root/reference/pkg/src, plus its tests/support.py helpers),
solves every fixture LP with the reference's own ``solve`` / ``batch_solve``,
and writes:

  known.json    hand-built known-answer LPs (the reference's test LPs and
                edge shapes) with their limits and reference outcomes
  ragged.json   seeded random families of varying shape (the reference's
                acceptance / simplex test families plus mixed-sign and
                degenerate families)
  <cfg>.npz     packed same-shape families per kernel variant; inputs are
                regenerated from the committed recipe in
                paper_1802_08557_b200/workloads.py and pinned by sha256.

Outcome encoding: status code (0 optimal, 1 unbounded, 2 infeasible,
3 iteration_limit), objective (NaN unless optimal), x (zeros unless
optimal), iterations per phase.  Floats in JSON use repr (round-trips).
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, str(REPO))

import batchlp  # noqa: E402  (the reference)
import support  # noqa: E402  (the reference's test helpers)
from batchlp import BatchConfig, SolverLimits, StandardFormLP, batch_solve, solve, standard_form  # noqa: E402

from paper_1802_08557_b200 import workloads  # noqa: E402  (recipes only)

CODES = {"optimal": 0, "unbounded": 1, "infeasible": 2, "iteration_limit": 3}


def outcome_record(out) -> dict:
    rec = dict(status=CODES[out.status.value], it1=out.iterations_phase1, it2=out.iterations_phase2)
    if out.status.value == "optimal":
        rec["objective"] = float(out.objective_value)
        rec["x"] = [float(v) for v in out.primal_point]
    return rec


def lp_record(name, lp, limits: SolverLimits) -> dict:
    out = solve(lp, limits)
    return dict(name=name, m=lp.m, n=lp.n, A=np.asarray(lp.A, float).reshape(lp.m, lp.n).tolist(),
                b=[float(v) for v in lp.b], c=[float(v) for v in lp.c],
                limits=dict(max_iterations=limits.max_iterations, anti_cycling=limits.anti_cycling,
                            degenerate_pivot_limit=limits.degenerate_pivot_limit),
                outcome=outcome_record(out))


BEALE = standard_form([0.75, -150.0, 0.02, -6.0],
                      [[0.25, -60.0, -0.04, 9.0], [0.5, -90.0, -0.02, 3.0], [0.0, 0.0, 1.0, 0.0]],
                      [0.0, 0.0, 1.0])
WORKSHOP = standard_form([3.0, 5.0], [[1, 0], [0, 2], [3, 2]], [4.0, 12.0, 18.0])


def known_lps():
    L = SolverLimits
    cases = [
        ("workshop", WORKSHOP, L()),                                                   # test_simplex.py:17-24
        ("workshop_max_iter_1", WORKSHOP, L(max_iterations=1)),                        # :38-41
        ("unbounded", standard_form([1.0, 1.0], [[-1.0, 1.0]], [1.0]), L()),           # :27-30
        ("infeasible_phase1", standard_form([1.0], [[1.0]], [-1.0]), L()),             # :33-35
        ("single_negated_row", standard_form([1.0], [[2.0]], [-3.0]), L()),            # :55-60
        ("two_negated_rows", standard_form([1.0, 1.0], [[1.0, 0.0], [0.0, 1.0]], [-2.0, -5.0]), L()),
        ("equality_pair", standard_form([1.0, 0.0], [[1.0, 1.0], [-1.0, -1.0]], [2.0, -2.0]), L()),  # :87-109
        ("redundant_rows", standard_form([1.0, 1.0], [[1.0, 1.0], [-1.0, -1.0], [1.0, 1.0], [-1.0, -1.0]],
                                         [2.0, -2.0, 2.0, -2.0]), L()),               # :111-121
        ("beale", BEALE, L()),                                                         # :168-182
        ("beale_no_anticycling", BEALE, L(anti_cycling=False, max_iterations=200)),    # :184-186
        ("beale_trigger_0", BEALE, L(degenerate_pivot_limit=0)),
        ("beale_trigger_1", BEALE, L(degenerate_pivot_limit=1)),
        ("beale_trigger_5", BEALE, L(degenerate_pivot_limit=5)),
        ("small_single_pivot", standard_form([3.0], [[1.0]], [4.0]), L()),             # test_tableau.py:21-23
        ("zero_column_rows", standard_form([2.0, 1.0], [[1.0, 0.0], [0.0, 1.0]], [3.0, 5.0]), L()),
        ("no_rows_unbounded", StandardFormLP(c=np.array([1.0, 2.0]), A=np.zeros((0, 2)), b=np.zeros(0)), L()),
        ("no_rows_optimal", StandardFormLP(c=np.array([-1.0, 0.0]), A=np.zeros((0, 2)), b=np.zeros(0)), L()),
        ("no_cols_feasible", StandardFormLP(c=np.zeros(0), A=np.zeros((2, 0)), b=np.array([1.0, 2.0])), L()),
        ("no_cols_infeasible", StandardFormLP(c=np.zeros(0), A=np.zeros((2, 0)), b=np.array([1.0, -2.0])), L()),
        ("zero_objective", standard_form([0.0, 0.0], [[1.0, 2.0], [3.0, 1.0]], [4.0, 5.0]), L()),
        ("degenerate_zero_rhs", standard_form([1.0, 1.0], [[1.0, -1.0], [-1.0, 1.0], [1.0, 1.0]],
                                              [0.0, 0.0, 2.0]), L()),
        ("mixed_phase1_limit", standard_form([1.0, 2.0], [[1.0, 1.0], [-1.0, -2.0], [2.0, -1.0]],
                                             [4.0, -2.0, 3.0]), L(max_iterations=1)),
        ("negative_zero_b", standard_form([1.0], [[1.0]], [-0.0]), L()),
        ("fractional", standard_form([0.1, 0.7, 0.3], [[0.3, 0.9, 0.2], [0.7, 0.1, 0.8]], [1.1, 0.7]), L()),
        ("huge_coeffs", standard_form([1e150, 1.0], [[1e-150, 1.0], [1.0, 1e150]], [1e150, 1e-150]), L()),
    ]
    return [lp_record(name, lp, lim) for name, lp, lim in cases]


def ragged_lps():
    recs = []
    rng = np.random.default_rng(202401)                      # test_acceptance.py:49-65
    for k in range(300):
        recs.append(lp_record(f"crit1_{k}", support.random_lp(rng, (2, 7), (3, 9), 1, 101), SolverLimits()))
    rng = np.random.default_rng(202402)                      # test_acceptance.py:68-82
    for k in range(100):
        recs.append(lp_record(f"crit2_{k}", support.random_lp(rng, (2, 7), (3, 9), 1, 101, negate_b=True),
                              SolverLimits()))
    rng = np.random.default_rng(21)                          # test_simplex.py:124-145
    for k in range(120):
        n = int(rng.integers(2, 6))
        m = int(rng.integers(2, 7))
        A = rng.integers(-50, 51, size=(m, n)).astype(float)
        x0 = rng.integers(1, 5, size=n).astype(float)
        b = A @ x0 + rng.integers(1, 20, size=m).astype(float)
        c = rng.integers(1, 51, size=n).astype(float)
        recs.append(lp_record(f"mixed21_{k}", standard_form(c, A, b), SolverLimits()))
    rng = np.random.default_rng(90001)                       # mixed signs: all four statuses
    for k in range(400):
        n = int(rng.integers(1, 13))
        m = int(rng.integers(1, 13))
        A = rng.integers(-9, 10, size=(m, n)).astype(float)
        b = rng.integers(-20, 41, size=m).astype(float)
        c = rng.integers(-5, 11, size=n).astype(float)
        recs.append(lp_record(f"signs_{k}", standard_form(c, A, b), SolverLimits()))
    rng = np.random.default_rng(90002)                       # degenerate: zero rhs, Bland switches
    for k in range(300):
        n = int(rng.integers(2, 10))
        m = int(rng.integers(2, 10))
        A = rng.integers(-2, 3, size=(m, n)).astype(float)
        b = rng.integers(-1, 2, size=m).astype(float)
        c = rng.integers(-2, 4, size=n).astype(float)
        lim = SolverLimits(degenerate_pivot_limit=int(rng.integers(0, 3))) if k % 3 == 0 else SolverLimits()
        recs.append(lp_record(f"degen_{k}", standard_form(c, A, b), lim))
    rng = np.random.default_rng(90003)                       # fractional coefficients
    for k in range(200):
        n = int(rng.integers(2, 9))
        m = int(rng.integers(2, 9))
        A = rng.uniform(-1, 1, size=(m, n)).round(3)
        b = rng.uniform(-0.5, 2, size=m).round(3)
        c = rng.uniform(-1, 1, size=n).round(3)
        recs.append(lp_record(f"frac_{k}", standard_form(c, A, b), SolverLimits()))
    return recs


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def solve_packed(A, b, c, shared=False, workers=8, limits=SolverLimits()):
    count = len(c)
    lps = [StandardFormLP(c=c[k], A=A if shared else A[k], b=b if shared else b[k]) for k in range(count)]
    rep = batch_solve(lps, BatchConfig(worker_count=workers, limits=limits))
    n = c.shape[1]
    status = np.array([CODES[o.status.value] for o in rep.outcomes], np.int8)
    obj = np.array([o.objective_value if o.objective_value is not None else np.nan for o in rep.outcomes])
    x = np.array([o.primal_point if o.primal_point is not None else np.zeros(n) for o in rep.outcomes])
    it1 = np.array([o.iterations_phase1 for o in rep.outcomes], np.int32)
    it2 = np.array([o.iterations_phase2 for o in rep.outcomes], np.int32)
    return status, obj, x.reshape(count, n), it1, it2


# (file stem, recipe call as text, generator) -- the recipe text is stored in the fixture
PACKED = [
    ("c1_rand5", "workloads.random_arrays(5, 1000, 0)", lambda: (*workloads.random_arrays(5, 1000, 0), False)),
    ("c1_rand5_infeasible", "workloads.random_arrays(5, 200, 7, False)",
     lambda: (*workloads.random_arrays(5, 200, 7, False), False)),
    ("c2_afiro", "workloads.afiro_arrays(2000)", lambda: (*workloads.afiro_arrays(2000), False)),
    ("afiro_m12_n8", "workloads.afiro_arrays(1500, 11, 12, 8)",
     lambda: (*workloads.afiro_arrays(1500, 11, 12, 8), False)),
    ("afiro_m45_n30", "workloads.afiro_arrays(400, 12, 45, 30)",
     lambda: (*workloads.afiro_arrays(400, 12, 45, 30), False)),
    ("afiro_m20_n400", "workloads.afiro_arrays(60, 13, 20, 400)",
     lambda: (*workloads.afiro_arrays(60, 13, 20, 400), False)),
    ("c3_degenerate", "workloads.degenerate_arrays(400)", lambda: (*workloads.degenerate_arrays(400), False)),
    ("c3_beale", "workloads.padded_beale(100, 100)",
     lambda: tuple(np.asarray(v)[None] for v in workloads.padded_beale(100, 100)) + (False,)),
    ("c4_support", "workloads.support_polytope(); workloads.support_directions(2000)",
     lambda: (*workloads.support_polytope(), workloads.support_directions(2000), True)),
    ("afiro_m150_n150", "workloads.afiro_arrays(16, 14, 150, 150)",
     lambda: (*workloads.afiro_arrays(16, 14, 150, 150), False)),
    ("c5b_afiro500", "workloads.afiro_arrays(2, 55, 500, 500)",
     lambda: (*workloads.afiro_arrays(2, 55, 500, 500), False)),
    ("c5_rand500", "workloads.random_arrays(500, 3, 5)", lambda: (*workloads.random_arrays(500, 3, 5), False)),
]


def main(only=None):
    t0 = time.time()
    if only is None or "known" in only:
        (HERE / "known.json").write_text(json.dumps(known_lps(), indent=0))
        print("known.json", time.time() - t0, flush=True)
    if only is None or "ragged" in only:
        (HERE / "ragged.json").write_text(json.dumps(ragged_lps()))
        print("ragged.json", time.time() - t0, flush=True)
    for stem, recipe, gen in PACKED:
        if only is not None and stem not in only:
            continue
        A, b, c, shared = gen()
        status, obj, x, it1, it2 = solve_packed(A, b, c, shared)
        np.savez_compressed(HERE / f"{stem}.npz", recipe=recipe, sha256=sha(A, b, c), shared=shared,
                            m=b.shape[-1], n=c.shape[1], status=status, objective=obj, x=x, it1=it1, it2=it2,
                            reference=f"batchlp {batchlp.__version__} numpy {np.__version__}")
        print(stem, dict(zip(*np.unique(status, return_counts=True))), "pivots",
              float((it1 + it2).mean()), time.time() - t0, flush=True)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)


def box_records():
    """Hyper-rectangle LPs through the reference's solve_box (boxlp.py:44-61)."""
    from batchlp import BoxLP, InvalidBox, solve_box
    recs = []

    def add(name, lo, hi, d):
        box = BoxLP(np.asarray(lo, float), np.asarray(hi, float), np.asarray(d, float))
        try:
            sol = solve_box(box)
            out = dict(value=float(sol.value), point=[float(v) for v in sol.point])
        except InvalidBox as err:
            out = dict(error=str(err))
        recs.append(dict(name=name, lower=[float(v) for v in box.lower], upper=[float(v) for v in box.upper],
                         direction=[float(v) for v in box.direction], outcome=out))

    rng = np.random.default_rng(202403)                   # test_acceptance.py:85-95
    for k in range(300):
        n = int(rng.integers(1, 13))
        lower = rng.uniform(-10, 5, n)
        add(f"crit3_{k}", lower, lower + rng.uniform(0, 10, n), rng.uniform(-5, 5, n))
    add("zero_direction_takes_upper", [0.0, -1.0], [2.0, 3.0], [0.0, 0.0])
    add("negative_direction_takes_lower", [1.0, -4.0], [2.0, 3.0], [-1.0, -2.0])
    add("degenerate_box", [1.0, 1.0], [1.0, 1.0], [3.0, -3.0])
    add("lower_above_upper", [0.0, 5.0, 1.0], [1.0, 4.0, 0.0], [1.0, 1.0, 1.0])
    add("infinite_bound", [0.0, -np.inf], [1.0, 1.0], [1.0, 1.0])
    add("nan_bound", [0.0, np.nan], [1.0, 1.0], [1.0, 1.0])
    add("overflowing_sum", [1e308, 0.0], [1.7e308, 1.0], [1.0, 1.0])
    add("empty", [], [], [])
    return recs


def write_box():
    (HERE / "box.json").write_text(json.dumps(box_records(), allow_nan=True))
