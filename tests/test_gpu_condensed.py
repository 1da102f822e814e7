"""The condensed-tableau kernel family (blp_condensed_kernel.cuh: only the nonbasic
columns + rhs stored and updated) against the oracle and the reference goldens, on
every instance shape, two-phase LPs included (artificial/slack pairs, restore
pivots on the trivial slack, infeasible and phase-1 iteration limits).

Bar: status, x and per-phase iteration counts identical; objective within 1e-9
true relative error.
"""
import numpy as np
import pytest

from golden_io import compare, json_records, packed_fixture, packed_names

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture
def condensed(monkeypatch):
    monkeypatch.setenv("BLP_KERNEL", "condensed")
    yield


def _d(res):
    return dict(status=res.status, objective=res.objective, x=res.x, it1=res.iterations_phase1,
                it2=res.iterations_phase2)


def _mix(m, n, seed, count=240):
    """Two-phase afiro-style LPs (mixed-sign b, infeasible rows), the degenerate /
    unbounded / padded-Beale recipe, the reference's random generator, and equality-like
    pairs (a row and its negation: phase 1 ends with artificials basic at zero level)."""
    from paper_1802_08557_b200 import workloads
    if m >= 3 and n >= 4:
        A1, b1, c1 = workloads.afiro_arrays(count, seed=seed, m=m, n=n)
        A2, b2, c2 = workloads.degenerate_arrays(count, seed=seed + 1, m=m, n=n)
    else:   # tiny shapes: mixed-sign random LPs instead of the recipes (which need m >= 3, n >= 4)
        g = np.random.default_rng(seed)
        A1 = g.integers(-9, 10, size=(2 * count, m, n)).astype(np.float64)
        b1 = g.integers(-9, 10, size=(2 * count, m)).astype(np.float64)
        c1 = g.integers(-9, 10, size=(2 * count, n)).astype(np.float64)
        A2, b2, c2 = A1[:0], b1[:0], c1[:0]
    A3, b3, c3 = workloads.random_arrays(max(m, n), count // 4, seed + 2)
    A3, b3, c3 = A3[:, :m, :n], b3[:, :m], c3[:, :n]
    rng = np.random.default_rng(seed + 3)
    A4 = rng.integers(-5, 6, size=(count // 2, m, n)).astype(np.float64)
    x0 = rng.integers(0, 3, size=(count // 2, n)).astype(np.float64)
    b4 = np.einsum("kij,kj->ki", A4, x0)
    if m >= 2:
        h = m // 2
        A4[:, h:2 * h] = -A4[:, :h]            # A_h x <= b_h and -A_h x <= -b_h: equalities
        b4[:, h:2 * h] = -b4[:, :h]
    c4 = rng.integers(-4, 5, size=(count // 2, n)).astype(np.float64)
    A = np.ascontiguousarray(np.concatenate([A1, A2, A3, A4]))
    b = np.ascontiguousarray(np.concatenate([b1, b2, b3, b4]))
    c = np.ascontiguousarray(np.concatenate([c1, c2, c3, c4]))
    return A, b, c


SHAPES = [(1, 1), (2, 3), (5, 5), (8, 8), (12, 19), (28, 32), (30, 31), (32, 32), (32, 9), (20, 40), (31, 64),
          (33, 20), (40, 16), (64, 32), (64, 8), (50, 30), (65, 8), (100, 16), (128, 16), (90, 7)]


@pytest.mark.parametrize("cm", ["0", "3"])
@pytest.mark.parametrize("m,n", SHAPES)
def test_condensed_matches_oracle(m, n, cm, condensed, monkeypatch):
    """Every shape through the one-warp form (BLP_CMULTI=0) and, for 33..128 rows, the
    multi-warp form (BLP_CMULTI=3, blp_cmulti_kernel.cuh) too."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, batch_solve_arrays
    monkeypatch.setenv("BLP_CMULTI", cm)
    if cm == "3" and m <= 32:
        pytest.skip("the multi-warp form starts at 33 rows")
    variant = _native.kernel_variant(m, n)
    assert variant.startswith("cm" if cm == "3" else "ctab"), variant
    A, b, c = _mix(m, n, seed=m * 1000 + n)
    want = oracle.solve_batch(A, b, c)
    compare(_d(batch_solve_arrays(A, b, c)), want, f"{variant} {m}x{n}")


MULTI_SHAPES = [(33, 64), (64, 50), (70, 60), (100, 100), (99, 105), (120, 101), (128, 128), (65, 128),
                (129, 60), (150, 150), (180, 40), (200, 120), (256, 200), (256, 64),
                (257, 72), (300, 60), (450, 40), (512, 72)]


@pytest.mark.parametrize("m,n", MULTI_SHAPES)
def test_condensed_multiwarp_matches_oracle(m, n, condensed):
    """Shapes only the multi-warp form holds (n beyond the one-warp register rows; 129..256
    rows: eight row-warps), default dispatch: register slots + the shared-memory tile slots."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, batch_solve_arrays
    variant = _native.kernel_variant(m, n)
    assert variant.startswith("cm"), variant
    A, b, c = _mix(m, n, seed=m * 1000 + n, count=120 if m <= 128 else (40 if m <= 256 else 16))
    want = oracle.solve_batch(A, b, c, threads=oracle.host_cores())
    compare(_d(batch_solve_arrays(A, b, c)), want, f"{variant} {m}x{n}")


@pytest.mark.parametrize("m,n", [(12, 19), (28, 32), (64, 32), (100, 16)])
def test_condensed_solver_limits(m, n, condensed):
    from oracle import oracle
    from paper_1802_08557_b200 import SolverLimits, batch_solve_arrays
    A, b, c = _mix(m, n, seed=7 * m + n, count=120)
    for kw in (dict(max_iterations=1), dict(max_iterations=7), dict(degenerate_pivot_limit=0),
               dict(degenerate_pivot_limit=2), dict(anti_cycling=False, max_iterations=300)):
        want = oracle.solve_batch(A, b, c, **kw)
        compare(_d(batch_solve_arrays(A, b, c, SolverLimits(**kw))), want, f"ctab {m}x{n} {kw}")


def test_condensed_reference_records(condensed):
    """Every known-answer / ragged reference record whose shape the family covers."""
    from paper_1802_08557_b200 import SolverLimits, _native, batch_solve_arrays
    checked = 0
    for fixture in ("known.json", "ragged.json"):
        for rec in json_records(fixture):
            if not _native.kernel_variant(rec["m"], rec["n"]).startswith(("ctab", "cm")):
                continue
            res = batch_solve_arrays(rec["A"][None], rec["b"][None], rec["c"][None], SolverLimits(**rec["limits"]))
            o = rec["outcome"]
            want = dict(status=[o["status"]], it1=[o["it1"]], it2=[o["it2"]],
                        objective=[o.get("objective", np.nan)], x=[o.get("x", [0.0] * rec["n"])])
            compare(_d(res), want, f"{fixture}:{rec['name']}")
            checked += 1
    assert checked > 500


@pytest.mark.parametrize("stem", packed_names())
def test_condensed_packed_goldens(stem, condensed):
    from paper_1802_08557_b200 import _native, batch_solve_arrays, support_batch
    fx = packed_fixture(stem)
    m, n = fx["b"].shape[-1], fx["c"].shape[1]
    if not _native.kernel_variant(m, n, fx["shared"]).startswith(("ctab", "cm")):
        pytest.skip(f"{m}x{n} outside the condensed family")
    res = support_batch(fx["A"], fx["b"], fx["c"]) if fx["shared"] else batch_solve_arrays(fx["A"], fx["b"], fx["c"])
    compare(_d(res), fx, stem)


def test_condensed_support_two_phase(condensed):
    """Support mode on a polytope with negative b rows (phase 1 per direction)."""
    from oracle import oracle
    from paper_1802_08557_b200 import support_batch, workloads
    A, b = workloads.support_polytope()
    b = b.copy()
    A = A.copy()
    A[40:50] = -np.abs(A[40:50])
    b[40:50] = -0.05                      # -|a|.x <= -0.05: needs phase 1, still feasible
    C = workloads.support_directions(20_000, offset=77)
    want = oracle.solve_batch(A, b, C, shared_Ab=True)
    assert (want["it1"] > 0).all()
    compare(_d(support_batch(A, b, C)), want, "ctab support two-phase")


def test_condensed_non_finite_flags(condensed):
    from paper_1802_08557_b200 import _native, workloads
    A, b, c = workloads.afiro_arrays(64, seed=3)
    A[3, 27, 31] = np.nan
    b[5, 0] = np.inf
    c[9, 31] = -np.inf
    got = _native.solve_host(A, b, c, _native.make_limits())
    assert (got["status"][[3, 5, 9]] == 5).all()
    assert (np.delete(got["status"], [3, 5, 9]) != 5).all()


STAGE_SHAPES = [(1, 2), (5, 6), (12, 19), (28, 32), (30, 31), (32, 32), (20, 40), (31, 64), (40, 16), (64, 32),
                (100, 16)]


@pytest.mark.parametrize("stage", ["0", "2"])
@pytest.mark.parametrize("m,n", STAGE_SHAPES)
def test_condensed_tma_staging(m, n, stage, condensed, monkeypatch):
    """The one-warp kernel with its TMA staging of the next LP's A (BLP_CT_STAGE=2: one
    cp.async.bulk per row into shared memory, mbarrier completion) and without it (0): the
    same results as the oracle; odd n (rows not 16-byte multiples) falls back in-kernel."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, batch_solve_arrays
    monkeypatch.setenv("BLP_CMULTI", "0")
    monkeypatch.setenv("BLP_CT_STAGE", stage)
    variant = _native.kernel_variant(m, n)
    assert variant.startswith("ctab"), variant
    A, b, c = _mix(m, n, seed=m * 997 + n, count=160)
    want = oracle.solve_batch(A, b, c)
    compare(_d(batch_solve_arrays(A, b, c)), want, f"{variant} {m}x{n} stage={stage}")
    A[7, m - 1, n - 1] = np.nan      # validation is fused into the (staged) build
    got = _native.solve_host(A, b, c, _native.make_limits())
    assert got["status"][7] == 5
    assert np.array_equal(np.delete(got["status"], 7), np.delete(want["status"], 7))


def test_condensed_tma_staging_unaligned_device_pointer(condensed, monkeypatch):
    """A caller's device A that is only 8-byte aligned (a view one double into a buffer):
    the kernel must not issue bulk copies from it (16-byte alignment) and still match."""
    from oracle import oracle
    from paper_1802_08557_b200 import SolverLimits, _native, workloads
    monkeypatch.setenv("BLP_CT_STAGE", "2")
    A, b, c = workloads.afiro_arrays(300, seed=5, m=28, n=32)
    want = oracle.solve_batch(A, b, c)
    dev = torch.device("cuda:0")
    buf = torch.zeros(A.size + 1, dtype=torch.float64, device=dev)
    buf[1:] = torch.from_numpy(A.reshape(-1)).to(dev)
    tA = buf[1:].view(A.shape)
    assert tA.data_ptr() % 16 == 8
    tb, tc = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (b, c))
    cnt, nn = c.shape
    out = dict(status=torch.empty(cnt, dtype=torch.int8, device=dev),
               objective=torch.empty(cnt, dtype=torch.float64, device=dev),
               x=torch.empty(cnt, nn, dtype=torch.float64, device=dev),
               it1=torch.empty(cnt, dtype=torch.int32, device=dev),
               it2=torch.empty(cnt, dtype=torch.int32, device=dev))
    _native.solve_device(tA, tb, tc, SolverLimits().to_native(), out)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items()}
    compare(got, want, "ctab 28x32 unaligned A")
