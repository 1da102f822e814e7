"""Shared phase 1 in support-function mode (one A, b; many objective directions).

Phase 1 and restore_objective depend only on A and b (/root/reference/pkg/src/batchlp/
simplex.py:94-130,168-178), so the condensed kernels run them once per
batch (condensed_phase1_kernel) and start every direction from the restored tableau with its
own price-out.  The oracle solves every direction from scratch -- full phase 1 each time --
so equality here checks the sharing bitwise: status, x, both iteration counts.
"""
import numpy as np
import pytest

from golden_io import compare

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _d(res):
    return dict(status=res["status"], objective=res["objective"], x=res["x"], it1=res["it1"], it2=res["it2"])


def _solve(A, b, C, **lim):
    from paper_1802_08557_b200 import _native
    return _native.solve_host(np.ascontiguousarray(A), np.ascontiguousarray(b), np.ascontiguousarray(C),
                              _native.make_limits(**lim), shared_Ab=True)


def test_c4b_directions_match_oracle():
    from oracle import oracle
    from paper_1802_08557_b200 import _native, workloads
    A, b = workloads.support_polytope_two_phase()
    C = workloads.support_directions(20_000)
    assert (b < 0).sum() == 16
    assert _native.kernel_variant(64, 32, True).startswith(("ctab", "cm"))
    got = _solve(A, b, C)
    want = oracle.solve_batch(A, b, C, shared_Ab=True, threads=oracle.host_cores())
    compare(_d(got), want, "c4b 20k directions")
    assert (got["it1"] == want["it1"][0]).all() and want["it1"][0] > 0


@pytest.mark.parametrize("cm", ["0", "3"])
@pytest.mark.parametrize("m,n", [(20, 12), (28, 32), (40, 16), (64, 8), (100, 12), (64, 32), (100, 100), (120, 128),
                                 (160, 48), (220, 150), (400, 60)])
def test_shared_phase1_every_condensed_shape(m, n, cm, monkeypatch):
    """Every condensed instance family -- one warp (rows per lane 1/2/4; BLP_CMULTI=0) and
    multi-warp (cmulti, registers + tile; BLP_CMULTI=3) -- with a mixed-sign shared b:
    afiro-recipe polytopes, feasible and infeasible, random directions."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, workloads
    monkeypatch.setenv("BLP_CMULTI", cm)
    variant = _native.kernel_variant(m, n, True)
    if not variant.startswith(("ctab", "cm")):
        pytest.skip(f"{m}x{n}: no one-warp instance")
    assert variant.startswith("cm" if cm == "3" and m > 32 else "ctab"), variant
    for seed in range(4):
        A, b, _ = workloads.afiro_arrays(1, seed=100 + seed, m=m, n=n, infeasible_frac=0.5)
        C = np.random.default_rng(seed).integers(-20, 51, size=(300, n)).astype(np.float64)
        got = _solve(A[0], b[0], C)
        want = oracle.solve_batch(A[0], b[0], C, shared_Ab=True)
        compare(_d(got), want, f"shared phase 1 {m}x{n} seed {seed}")


def test_infeasible_polytope_every_direction():
    from oracle import oracle
    from paper_1802_08557_b200 import workloads
    A, b = workloads.support_polytope_two_phase()
    A[40] = -A[0]
    b[40] = -b[0] - 1.0
    C = workloads.support_directions(500)
    got = _solve(A, b, C)
    want = oracle.solve_batch(A, b, C, shared_Ab=True)
    compare(_d(got), want, "infeasible polytope")
    assert (got["status"] == 2).all() and (got["it2"] == 0).all()


@pytest.mark.parametrize("lim", [dict(max_iterations=3), dict(max_iterations=20), dict(anti_cycling=False),
                                 dict(degenerate_pivot_limit=1)])
def test_limits_flow_through_shared_phase1(lim):
    from oracle import oracle
    from paper_1802_08557_b200 import workloads
    A, b = workloads.support_polytope_two_phase()
    C = workloads.support_directions(2000)
    got = _solve(A, b, C, **lim)
    want = oracle.solve_batch(A, b, C, shared_Ab=True, **lim)
    compare(_d(got), want, f"shared phase 1 limits {lim}")


def test_non_finite_direction_and_polytope():
    from paper_1802_08557_b200 import workloads
    from oracle import oracle
    A, b = workloads.support_polytope_two_phase()
    C = workloads.support_directions(64)
    C[5, 3] = np.nan
    C[17, 31] = np.inf
    got = _solve(A, b, C)
    assert (got["status"][[5, 17]] == 5).all()
    ok = [k for k in range(64) if k not in (5, 17)]
    want = oracle.solve_batch(A, b, C[ok], shared_Ab=True)
    for key in ("status", "it1", "it2", "x"):
        assert np.array_equal(got[key][ok], want[key]), key
    A2 = A.copy()
    A2[50, 7] = np.inf
    assert (_solve(A2, b, C)["status"] == 5).all()
    b2 = b.copy()
    b2[33] = np.nan
    assert (_solve(A, b2, C)["status"] == 5).all()


def test_support_batch_api_two_phase_and_sub_batches(monkeypatch):
    """The public support_batch over many host sub-batches (each re-runs the prologue)."""
    from oracle import oracle
    from paper_1802_08557_b200 import support_batch, workloads
    monkeypatch.setenv("BLP_HOST_CHUNKS", "7")
    A, b = workloads.support_polytope_two_phase()
    C = workloads.support_directions(30_001)
    got = support_batch(A, b, C)
    want = oracle.solve_batch(A, b, C, shared_Ab=True, threads=oracle.host_cores())
    compare(dict(status=got.status, objective=got.objective, x=got.x, it1=got.iterations_phase1,
                 it2=got.iterations_phase2), want, "support_batch two-phase")
