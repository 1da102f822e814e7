"""The CPU oracle (oracle/blp_oracle.c) against every golden fixture the reference produced.

This pins the oracle before it is trusted as the checker of the CUDA path:
status, x and per-phase iteration counts must equal the reference's exactly,
the objective within 1e-9 relative (the reference's c.x is a BLAS ddot).
"""
import numpy as np
import pytest

from golden_io import compare, json_records, packed_fixture, packed_names
from oracle import oracle


def _want(rec):
    o = rec["outcome"]
    n = rec["n"]
    return dict(status=[o["status"]], it1=[o["it1"]], it2=[o["it2"]],
                objective=[o.get("objective", np.nan)], x=[o.get("x", [0.0] * n)] if n else np.zeros((1, 0)))


@pytest.mark.parametrize("fixture", ["known.json", "ragged.json"])
def test_oracle_matches_reference_records(fixture):
    for rec in json_records(fixture):
        got = oracle.solve_batch(rec["A"][None], rec["b"][None], rec["c"][None], threads=1, **rec["limits"])
        compare(got, _want(rec), f"{fixture}:{rec['name']}")


@pytest.mark.parametrize("stem", packed_names())
def test_oracle_matches_reference_packed(stem):
    fx = packed_fixture(stem)
    got = oracle.solve_batch(fx["A"], fx["b"], fx["c"], shared_Ab=fx["shared"])
    compare(got, fx, stem)


def test_oracle_thread_count_does_not_change_results():
    fx = packed_fixture("c2_afiro")
    one = oracle.solve_batch(fx["A"][:300], fx["b"][:300], fx["c"][:300], threads=1)
    many = oracle.solve_batch(fx["A"][:300], fx["b"][:300], fx["c"][:300], threads=4)
    for k in ("status", "it1", "it2", "x"):
        assert np.array_equal(one[k], many[k])
    assert np.array_equal(one["objective"], many["objective"], equal_nan=True)


def test_oracle_against_live_reference(reference):
    """Fresh seeded LPs (not in the fixtures) solved by the imported reference and the oracle."""
    rng = np.random.default_rng(4242)
    for k in range(150):
        n = int(rng.integers(1, 9))
        m = int(rng.integers(0, 9))
        A = rng.integers(-6, 7, size=(m, n)).astype(float)
        b = rng.integers(-8, 20, size=m).astype(float)
        c = rng.integers(-4, 9, size=n).astype(float)
        out = reference.solve(reference.standard_form(c, A, b))
        got = oracle.solve_batch(A[None], b[None], c[None], threads=1)
        codes = {"optimal": 0, "unbounded": 1, "infeasible": 2, "iteration_limit": 3}
        want = dict(status=[codes[out.status.value]], it1=[out.iterations_phase1], it2=[out.iterations_phase2],
                    objective=[out.objective_value if out.objective_value is not None else np.nan],
                    x=[out.primal_point if out.primal_point is not None else np.zeros(n)])
        compare(got, want, f"live{k}")


def test_box_oracle_matches_reference():
    from golden_io import box_arrays, box_records, compare_box
    for rec in box_records():
        lo, hi, d = box_arrays(rec)
        r = oracle.box_solve(lo, hi, d)
        compare_box(r["value"][0], r["point"][0], r["status"][0], rec)
