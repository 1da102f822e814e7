"""CUDA path vs the reference (golden fixtures) and vs the CPU oracle -- through the C ABI.

Bar (BASELINE.json north star): status, x and per-phase iteration counts
identical to the reference; objective within 1e-9 relative.
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


def _native_dict(res):
    return dict(status=res.status, objective=res.objective, x=res.x, it1=res.iterations_phase1,
                it2=res.iterations_phase2)


def _want(rec):
    o = rec["outcome"]
    n = rec["n"]
    return dict(status=[o["status"]], it1=[o["it1"]], it2=[o["it2"]],
                objective=[o.get("objective", np.nan)], x=[o.get("x", [0.0] * n)] if n else np.zeros((1, 0)))


@pytest.mark.parametrize("fixture", ["known.json", "ragged.json"])
def test_records_match_reference(fixture):
    from paper_1802_08557_b200 import SolverLimits, batch_solve_arrays
    for rec in json_records(fixture):
        res = batch_solve_arrays(rec["A"][None], rec["b"][None], rec["c"][None], SolverLimits(**rec["limits"]))
        compare(_native_dict(res), _want(rec), f"{fixture}:{rec['name']}")


def test_records_batched_by_shape_match_reference():
    """Same records, grouped into same-shape batches (exercises the persistent LP queue)."""
    from paper_1802_08557_b200 import batch_solve_arrays
    groups = {}
    for rec in json_records("ragged.json"):
        if rec["limits"] == dict(max_iterations=None, anti_cycling=True, degenerate_pivot_limit=None):
            groups.setdefault((rec["m"], rec["n"]), []).append(rec)
    for shape, recs in groups.items():
        A = np.stack([r["A"] for r in recs]).reshape(len(recs), *shape)
        b = np.stack([r["b"] for r in recs]).reshape(len(recs), shape[0])
        c = np.stack([r["c"] for r in recs]).reshape(len(recs), shape[1])
        res = batch_solve_arrays(A, b, c)
        for k, r in enumerate(recs):
            got = {key: val[k:k + 1] for key, val in _native_dict(res).items()}
            compare(got, _want(r), f"{shape}:{r['name']}")


@pytest.mark.parametrize("stem", packed_names())
def test_packed_families_match_reference(stem):
    from paper_1802_08557_b200 import batch_solve_arrays, support_batch
    fx = packed_fixture(stem)
    if fx["shared"]:
        res = support_batch(fx["A"], fx["b"], fx["c"])
    else:
        res = batch_solve_arrays(fx["A"], fx["b"], fx["c"])
    compare(_native_dict(res), fx, stem)


def test_object_api_matches_reference_layout():
    """batch_solve / solve return SolveOutcome objects laid out as the reference's."""
    from paper_1802_08557_b200 import BatchConfig, Status, batch_solve, gen_random_lps, solve, standard_form
    lp = standard_form([3.0, 5.0], [[1, 0], [0, 2], [3, 2]], [4.0, 12.0, 18.0])
    out = solve(lp)
    assert out.status is Status.OPTIMAL and out.objective_value == pytest.approx(36.0)
    assert out.primal_point.tolist() == [2.0, 6.0]
    lps = gen_random_lps(5, 40, seed=11)
    rep = batch_solve(lps, BatchConfig(memory_budget_bytes=768 * 7))
    assert rep.plan.count == 6 and len(rep.chunk_seconds) == 6
    for lp_k, o in zip(lps, rep.outcomes):
        d = solve(lp_k)
        assert (o.status, o.objective_value, o.iterations_phase1, o.iterations_phase2) == \
            (d.status, d.objective_value, d.iterations_phase1, d.iterations_phase2)
        assert np.array_equal(o.primal_point, d.primal_point)
    assert rep.status_counts() == {"optimal": 40}


def test_invalid_lp_raises_reference_message():
    from paper_1802_08557_b200 import batch_solve, standard_form, solve
    with pytest.raises(ValueError, match="invalid LP: A\\[0\\]\\[0\\] is not finite"):
        solve(standard_form([1.0], [[np.nan]], [1.0]))
    lps = [standard_form([1.0], [[1.0]], [1.0]), standard_form([1.0], [[1.0]], [np.inf])]
    with pytest.raises(ValueError, match="invalid LP: b\\[0\\] is not finite"):
        batch_solve(lps)


def test_afiro_against_oracle_20k():
    """20,000 fresh C2-recipe LPs (seed not in the fixtures) vs the CPU oracle."""
    from oracle import oracle
    from paper_1802_08557_b200 import batch_solve_arrays, workloads
    A, b, c = workloads.afiro_arrays(20_000, seed=77)
    res = batch_solve_arrays(A, b, c)
    compare(_native_dict(res), oracle.solve_batch(A, b, c), "afiro20k")


def test_support_against_oracle_and_unshared():
    """Support-function mode equals the same LPs solved with A, b replicated."""
    from oracle import oracle
    from paper_1802_08557_b200 import batch_solve_arrays, support_batch, workloads
    A, b = workloads.support_polytope()
    C = workloads.support_directions(5000, offset=2000)
    res = support_batch(A, b, C)
    compare(_native_dict(res), oracle.solve_batch(A, b, C, shared_Ab=True), "support5k")
    rep = batch_solve_arrays(np.broadcast_to(A, (len(C),) + A.shape), np.broadcast_to(b, (len(C),) + b.shape), C)
    compare(_native_dict(rep), _native_dict(res), "support-vs-replicated")


def test_device_api_equals_host_api():
    """blp_solve_batch_device on torch tensors == blp_solve_batch_host on numpy arrays."""
    from paper_1802_08557_b200 import SolverLimits, _native, batch_solve_arrays, workloads
    A, b, c = workloads.afiro_arrays(3000, seed=5)
    host = _native_dict(batch_solve_arrays(A, b, c))
    dev = torch.device("cuda:0")
    tA, tb, tc = (torch.from_numpy(v).to(dev) for v in (A, b, c))
    out = dict(status=torch.empty(3000, dtype=torch.int8, device=dev),
               objective=torch.empty(3000, dtype=torch.float64, device=dev),
               x=torch.empty(3000, 32, dtype=torch.float64, device=dev),
               it1=torch.empty(3000, dtype=torch.int32, device=dev),
               it2=torch.empty(3000, dtype=torch.int32, device=dev))
    _native.solve_device(tA, tb, tc, SolverLimits().to_native(), out)
    torch.cuda.synchronize()
    compare({k: v.cpu().numpy() for k, v in out.items()}, host, "device-vs-host")


def test_full_size_c2_properties():
    """BASELINE size (1e5 C2 LPs): determinism, chunk invariance and certificate properties."""
    from paper_1802_08557_b200 import batch_solve_arrays, workloads
    A, b, c = workloads.afiro_arrays(100_000)
    r1 = batch_solve_arrays(A, b, c)
    r2 = batch_solve_arrays(A, b, c)
    compare(_native_dict(r1), _native_dict(r2), "determinism")
    half = batch_solve_arrays(A[50_000:], b[50_000:], c[50_000:])
    compare(_native_dict(half), {k: v[50_000:] for k, v in _native_dict(r1).items()}, "chunk-invariance")
    opt = r1.status == 0
    assert 0.85 < opt.mean() < 0.95 and set(np.unique(r1.status)) <= {0, 2}
    x = r1.x[opt]
    assert (x >= 0).all()
    slack = b[opt] - np.einsum("kij,kj->ki", A[opt], x)
    assert (slack >= -1e-6 * np.maximum(1, np.abs(b[opt]))).all()
    assert np.allclose(np.einsum("kj,kj->k", c[opt], x), r1.objective[opt], rtol=1e-12, atol=1e-9)
    # the infeasible recipe rows are exactly the infeasible outcomes
    assert (r1.status == 2).sum() > 5000


def test_c3_sample_against_oracle():
    """C3 recipe, 2000 fresh LPs (degenerate, unbounded, infeasible, Beale) vs the oracle."""
    from oracle import oracle
    from paper_1802_08557_b200 import batch_solve_arrays, workloads
    A, b, c = workloads.degenerate_arrays(2000, seed=33)
    res = batch_solve_arrays(A, b, c)
    compare(_native_dict(res), oracle.solve_batch(A, b, c), "c3-2000")
    assert set(np.unique(res.status)) == {0, 1, 2}


def test_iteration_limit_and_trigger_limits_flow_through():
    from oracle import oracle
    from paper_1802_08557_b200 import SolverLimits, batch_solve_arrays, workloads
    A, b, c = workloads.degenerate_arrays(300, seed=34)
    for lim in (dict(max_iterations=7), dict(degenerate_pivot_limit=0), dict(degenerate_pivot_limit=3),
                dict(anti_cycling=False, max_iterations=400)):
        res = batch_solve_arrays(A, b, c, SolverLimits(**lim))
        compare(_native_dict(res), oracle.solve_batch(A, b, c, **lim), f"limits {lim}")


def test_box_records_match_reference():
    """Batched hyper-rectangle LPs (the paper's Eq. 7 kernel) vs the reference's solve_box."""
    from golden_io import box_arrays, box_records, compare_box
    from paper_1802_08557_b200 import BoxLP, InvalidBox, box_batch_arrays, solve_box, solve_box_batch
    recs = box_records()
    for rec in recs:
        lo, hi, d = box_arrays(rec)
        r = box_batch_arrays(lo, hi, d)
        compare_box(r.value[0], r.point[0], r.status[0], rec)
    boxes = [BoxLP.build(r["lower"], r["upper"], r["direction"]) for r in recs]
    got = solve_box_batch(boxes)
    for rec, g in zip(recs, got):
        if "error" in rec["outcome"]:
            assert isinstance(g, InvalidBox) and str(g) == rec["outcome"]["error"]
        else:
            assert np.array_equal(g.point, np.asarray(rec["outcome"]["point"]))
    with pytest.raises(InvalidBox, match="box bounds must be finite"):
        solve_box(BoxLP.build([0.0], [np.inf], [1.0]))


def test_box_batch_1e5_against_oracle():
    """Criterion-3 batch shape: 1e5 boxes of dimension 5 (test_acceptance.py:96-104)."""
    from oracle import oracle
    from paper_1802_08557_b200 import box_batch_arrays
    rng = np.random.default_rng(77)
    lo = rng.uniform(-5, 5, (100_000, 5))
    hi = lo + rng.uniform(0, 5, (100_000, 5))
    d = rng.uniform(-3, 3, (100_000, 5))
    lo[17, 2], hi[17, 2] = 3.0, 1.0
    r = box_batch_arrays(lo, hi, d)
    w = oracle.box_solve(lo[:2000], hi[:2000], d[:2000])
    assert np.array_equal(r.status[:2000], w["status"]) and np.array_equal(r.point[:2000], w["point"])
    ok = w["status"] == 0
    assert np.allclose(r.value[:2000][ok], w["value"][ok], rtol=1e-12, atol=0)
    assert (r.status == 0).sum() == 100_000 - 1 and r.status[17] == 3


FAMILY_SHAPES = [(3, 5), (12, 19), (28, 32), (30, 31), (31, 32), (32, 32), (33, 20), (40, 50), (64, 33),
                 (64, 34), (65, 8), (100, 100), (128, 73), (128, 74), (90, 140), (100, 60), (120, 110),
                 (70, 128), (128, 128)]


@pytest.mark.parametrize("m,n", FAMILY_SHAPES)
def test_every_kernel_family_matches_oracle(m, n, monkeypatch):
    """Shapes on both sides of each kernel-family boundary, every applicable family forced
    (BLP_KERNEL / BLP_FORCE_HBM), each equal to the oracle: afiro-style two-phase LPs plus the
    degenerate / unbounded / infeasible / padded-Beale mix."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, batch_solve_arrays, workloads
    A1, b1, c1 = workloads.afiro_arrays(200, seed=m * 1000 + n, m=m, n=n)
    A2, b2, c2 = workloads.degenerate_arrays(300, seed=m * 1000 + n + 1, m=m, n=n)
    A, b, c = (np.concatenate(v) for v in ((A1, A2), (b1, b2), (c1, c2)))
    want = oracle.solve_batch(A, b, c)
    seen = set()
    for force, hbm, cm in (("", "0", "1"), ("condensed", "0", "0"), ("condensed", "0", "3"), ("warplp", "0", "1"),
                           ("pairlp", "0", "1"), ("regtile", "0", "1"), ("smem", "0", "1"), ("smem", "1", "1")):
        monkeypatch.setenv("BLP_KERNEL", force)
        monkeypatch.setenv("BLP_FORCE_HBM", hbm)
        monkeypatch.setenv("BLP_CMULTI", cm)
        variant = _native.kernel_variant(m, n)
        if variant in seen:
            continue
        seen.add(variant)
        res = batch_solve_arrays(A, b, c)
        compare(_native_dict(res), want, f"({m},{n}) {variant}")
    assert seen


@pytest.mark.filterwarnings("ignore::UserWarning")   # the edge-case MPS texts warn by design
def test_general_form_batches_match_reference():
    """General-form ingest (MPS fixtures + seeded general LPs) -> packed GPU batches per lowered
    shape -> recover_batch, vs the reference's standardize / solve / recover_outcome."""
    import json
    from golden_io import GOLDEN, obj_close
    from paper_1802_08557_b200 import GeneralLP, batch_solve_general, lower_to_general, parse_mps

    def glp_of(g):
        return GeneralLP.build(g["sense"], g["c"], np.asarray(g["rows"]).reshape(g["k"], g["n"]), g["relations"],
                               g["rhs"], g["lower"], g["upper"], g["row_names"], g["col_names"])

    items = []
    for r in json.loads((GOLDEN / "general.json").read_text())["records"]:
        if "error" not in r["lowered"]:
            items.append((r["name"], glp_of(r["general"]), r["lowered"]))
    for r in json.loads((GOLDEN / "mps.json").read_text())["records"]:
        if "lowered" in r and "error" not in r["lowered"]:
            items.append((r["name"], lower_to_general(parse_mps(r["text"])), r["lowered"]))
    groups = {}
    for it in items:
        groups.setdefault((it[2]["m"], it[2]["n"]), []).append(it)
    checked = 0
    for shape, group in groups.items():
        got = batch_solve_general([g for _, g, _ in group])
        for k, (name, _, want) in enumerate(group):
            w = want["outcome"]
            assert got.status[k] == w["status"], name
            assert (got.iterations_phase1[k], got.iterations_phase2[k]) == (want["std"]["it1"], want["std"]["it2"]), name
            if w["status"] == 0:
                assert np.array_equal(got.x[k], np.asarray(w["x"])), name
                assert obj_close(got.objective[k], w["objective"]), name
            checked += 1
    assert checked > 650


CLUSTER_CASES = [((45, 30), 2), ((45, 30), 3), ((45, 30), 16), ((100, 150), 0), ((100, 150), 5),
                 ((150, 150), 0), ((150, 150), 7), ((20, 400), 2), ((20, 400), 13), ((130, 90), 4),
                 ((300, 200), 0)]


@pytest.mark.parametrize("shape,K", CLUSTER_CASES)
def test_cluster_kernel_matches_oracle(shape, K, monkeypatch):
    """The cluster-resident variant (tableau split by columns over K CTAs, one DSMEM
    exchange per pivot) forced on shapes either side of its register/tile split,
    including K where a CTA owns fewer columns than its register half: equal to the oracle."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, batch_solve_arrays, workloads
    m, n = shape
    cnt = 60 if m * n > 20000 else 150
    A1, b1, c1 = workloads.afiro_arrays(cnt, seed=m * 1000 + n, m=m, n=n)
    A2, b2, c2 = workloads.degenerate_arrays(cnt, seed=m * 1000 + n + 1, m=m, n=n)
    A, b, c = (np.concatenate(v) for v in ((A1, A2), (b1, b2), (c1, c2)))
    want = oracle.solve_batch(A, b, c)
    monkeypatch.setenv("BLP_KERNEL", "cluster")
    monkeypatch.setenv("BLP_CLUSTER_K", str(K))
    monkeypatch.setenv("BLP_LAZY", "0")          # the dense cluster kernel for every LP
    assert _native.kernel_variant(m, n).startswith("cluster")
    res = batch_solve_arrays(A, b, c)
    compare(_native_dict(res), want, f"cluster {shape} K={K}")


LAZY_CASES = [(150, 150), (300, 200), (100, 150), (40, 300), (64, 30)]   # 500 x 500: the c5 goldens


def _single_phase_mix(m, n, seed):
    """Single-phase LPs (b >= 0): the C5 recipe, plus the degenerate/unbounded C3 recipe
    with |b| (zero rows of b make ties and Bland switches), plus long-running afiro-style
    LPs with |b| that exceed the lazy kernel's pivot budget and must be deferred."""
    from paper_1802_08557_b200 import workloads
    cnt = 24 if m * n > 100_000 else 80
    A1, b1, c1 = workloads.random_arrays(max(m, n), cnt, seed)
    A1, b1, c1 = A1[:, :m, :n].copy(), b1[:, :m].copy(), c1[:, :n].copy()
    A2, b2, c2 = workloads.degenerate_arrays(cnt, seed=seed + 1, m=m, n=n)
    A3, b3, c3 = workloads.afiro_arrays(cnt // 2, seed=seed + 2, m=m, n=n)
    A = np.concatenate([A1, A2, A3])
    b = np.abs(np.concatenate([b1, b2, b3]))
    c = np.concatenate([c1, c2, c3])
    return A, b, c


@pytest.mark.parametrize("sparse", ["1", "0"])
@pytest.mark.parametrize("m,n", LAZY_CASES)
def test_lazy_tableau_matches_oracle(m, n, sparse, monkeypatch):
    """The exact lazy-tableau kernel (entering column and pivot row evaluated by replaying
    the rank-1 update history) on single-phase LPs, with the cluster kernel taking the
    LPs it defers (phase 1 needed / more than 64 pivots): equal to the oracle, including
    iteration limits hit inside the lazy kernel.  BLP_LAZY_SPARSE=1 (opt-in, m >= 64): the
    slack columns of rows never pivoted on are skipped as exact unit columns."""
    from oracle import oracle
    from paper_1802_08557_b200 import SolverLimits, _native, batch_solve_arrays
    monkeypatch.setenv("BLP_LAZY_SPARSE", sparse)
    A, b, c = _single_phase_mix(m, n, seed=m * 7 + n)
    monkeypatch.setenv("BLP_KERNEL", "cluster")
    assert _native.kernel_variant(m, n).startswith("lazy")
    want = oracle.solve_batch(A, b, c)
    assert ((want["it1"] + want["it2"]) > 64).any() or m * n > 100_000
    compare(_native_dict(batch_solve_arrays(A, b, c)), want, f"lazy {m}x{n}")
    for mi in (1, 5, 40):
        want = oracle.solve_batch(A, b, c, max_iterations=mi)
        got = batch_solve_arrays(A, b, c, SolverLimits(max_iterations=mi))
        compare(_native_dict(got), want, f"lazy {m}x{n} max_iterations={mi}")


@pytest.mark.parametrize("split", ["1", "2"])
def test_lazy_split_mode_matches_oracle(split, monkeypatch):
    """BLP_LAZY_SPLIT=1|2 (validation as its own queue; half the CTAs or none validating
    first) on the single-phase mix, 150 x 150 and 100 x 100 (lazy ahead of cmulti): equal to
    the oracle."""
    from oracle import oracle
    from paper_1802_08557_b200 import batch_solve_arrays
    monkeypatch.setenv("BLP_LAZY_SPLIT", split)
    for m, n in ((150, 150), (100, 100)):
        A, b, c = _single_phase_mix(m, n, seed=m + 3)
        compare(_native_dict(batch_solve_arrays(A, b, c)), oracle.solve_batch(A, b, c), f"lazy split {m}x{n}")


def test_lazy_disabled_matches_lazy(monkeypatch):
    """BLP_LAZY=0 (dense cluster kernel for everything) gives the same bits."""
    from paper_1802_08557_b200 import batch_solve_arrays
    A, b, c = _single_phase_mix(150, 150, seed=5)
    r1 = _native_dict(batch_solve_arrays(A, b, c))
    monkeypatch.setenv("BLP_LAZY", "0")
    r2 = _native_dict(batch_solve_arrays(A, b, c))
    for k in r1:
        assert np.array_equal(r1[k], r2[k], equal_nan=True), k


@pytest.mark.parametrize("env", [{"BLP_LAZY_WS": "1"}, {"BLP_LAZY_WS": "1", "BLP_LAZY_PER_SM": "1"},
                                 {"BLP_LAZY_RP": "1"}, {"BLP_LAZY_NT": "256"}, {"BLP_LAZY_FSMEM": "1"}])
def test_lazy_kernel_forms_agree(monkeypatch, env):
    """The lazy kernel's alternative forms (warp-specialised bulk-copy validation
    stream, also with several LPs per CTA so the ring's mbarrier phases carry over
    between LPs; staged replay; CTA size) give the default form's bits, on an odd m*n
    (LPs alternate between 16-byte aligned and unaligned starts) with non-finite
    entries at the first and last element of A."""
    from paper_1802_08557_b200 import _native
    A, b, c = _single_phase_mix(151, 149, seed=8)
    A, b, c = np.tile(A, (4, 1, 1)), np.tile(b, (4, 1)), np.tile(c, (4, 1))   # more LPs than CTAs
    A[2, 0, 0] = np.nan
    A[5, 150, 148] = np.inf
    A[6, 150, 148] = -np.inf
    assert _native.kernel_variant(151, 149).startswith("lazy")
    lim = _native.make_limits()
    r1 = _native.solve_host(A, b, c, lim)
    assert (r1["status"][[2, 5, 6]] == 5).all()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    r2 = _native.solve_host(A, b, c, lim)
    for k in r1:
        assert np.array_equal(r1[k], r2[k], equal_nan=True), k


def test_lazy_support_staged_replay_matches_plain(monkeypatch):
    """Support mode runs the staged replay by default; the plain replay gives the same bits."""
    from paper_1802_08557_b200 import support_batch, workloads
    A, b = workloads.support_polytope()
    C = workloads.support_directions(4096)
    r1 = _native_dict(support_batch(A, b, C))
    monkeypatch.setenv("BLP_LAZY_RP", "0")
    r2 = _native_dict(support_batch(A, b, C))
    for k in r1:
        assert np.array_equal(r1[k], r2[k], equal_nan=True), k


@pytest.mark.parametrize("split", ["0", "1", "2"])
def test_lazy_path_flags_non_finite_entries(split, monkeypatch):
    """A non-finite entry anywhere in A (found by the concurrent validation pass -- inline, or
    the split mode's validation queue + finalize), b or c of a lazy-path batch: that LP comes
    back BLP_STATUS_INVALID, the others solved."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, workloads
    monkeypatch.setenv("BLP_LAZY_SPLIT", split)
    A, b, c = workloads.random_arrays(150, 12, seed=9)
    A[3, 149, 148] = np.nan
    A[5, 0, 0] = np.inf
    b[7, 10] = np.nan
    c[9, 149] = -np.inf
    assert _native.kernel_variant(150, 150).startswith("lazy")
    got = _native.solve_host(A, b, c, _native.make_limits())
    bad = [3, 5, 7, 9]
    assert (got["status"][bad] == 5).all()
    ok = [k for k in range(12) if k not in bad]
    want = oracle.solve_batch(A[ok], b[ok], c[ok])
    for key in ("status", "it1", "it2", "x"):
        assert np.array_equal(got[key][ok], want[key]), key


def test_lazy_support_mode_matches_oracle():
    """Support-function mode (one polytope, many objective directions) on a lazy-path
    shape, plus a non-finite polytope entry flagging every direction invalid."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, support_batch, workloads
    A, b, c = workloads.random_arrays(150, 1, seed=21)
    A, b = A[0], b[0]
    C = np.random.default_rng(22).normal(size=(300, 150))
    assert _native.kernel_variant(150, 150).startswith("lazy")
    got = support_batch(A, b, C)
    want = oracle.solve_batch(A, b, C, shared_Ab=True)
    compare(_native_dict(got), want, "lazy support 150x150")
    A2 = A.copy()
    A2[77, 3] = np.nan
    res = _native.solve_host(A2, b, C, _native.make_limits(), shared_Ab=True)
    assert (res["status"] == 5).all()


def test_lazy_ahead_of_hbm_kernel():
    """Beyond the cluster kernel's rows (m > 512) the lazy tableau runs ahead of the
    HBM-streamed kernel, which solves what it defers (here: phase-1 LPs)."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, batch_solve_arrays, workloads
    A, b, c = workloads.random_arrays(600, 10, seed=31)
    A2, b2, c2 = workloads.random_arrays(600, 3, seed=32, feasible_start=False)   # b < 0: phase 1, infeasible
    A, b, c = np.concatenate([A, A2]), np.concatenate([b, b2]), np.concatenate([c, c2])
    assert _native.kernel_variant(600, 600).startswith("lazy+hbm")
    got = batch_solve_arrays(A, b, c)
    compare(_native_dict(got), oracle.solve_batch(A, b, c), "lazy+hbm 600x600")
    assert (got.status[-3:] == 2).all()


@pytest.mark.parametrize("m,n", [(50, 50), (64, 64), (100, 100), (64, 40), (90, 150)])
def test_lazy_ahead_of_register_and_smem_kernels(m, n):
    """Default path for 33..128-row shapes: the lazy tableau takes the single-phase LPs, the
    pair/quad/smem kernel the ones it defers (phase 1, or > 64 pivots): equal to the oracle."""
    from oracle import oracle
    from paper_1802_08557_b200 import _native, batch_solve_arrays
    assert _native.kernel_variant(m, n).startswith("lazy+")
    A, b, c = _single_phase_mix(m, n, seed=m * 13 + n)
    from paper_1802_08557_b200 import workloads
    A2, b2, c2 = workloads.afiro_arrays(60, seed=m + n, m=m, n=n)           # two-phase: deferred at once
    A, b, c = np.concatenate([A, A2]), np.concatenate([b, b2]), np.concatenate([c, c2])
    want = oracle.solve_batch(A, b, c)
    compare(_native_dict(batch_solve_arrays(A, b, c)), want, f"lazy-first {m}x{n}")


def test_lazy_path_honours_solver_limits():
    """Limits flow through the lazy kernel exactly as through the dense ones: no
    anti-cycling, a custom degenerate-pivot trigger, small iteration caps."""
    from oracle import oracle
    from paper_1802_08557_b200 import SolverLimits, batch_solve_arrays
    A, b, c = _single_phase_mix(100, 100, seed=77)
    for kw in (dict(anti_cycling=False, max_iterations=30), dict(degenerate_pivot_limit=2),
               dict(degenerate_pivot_limit=1, max_iterations=50)):
        want = oracle.solve_batch(A, b, c, **kw)
        got = batch_solve_arrays(A, b, c, SolverLimits(**kw))
        compare(_native_dict(got), want, f"lazy limits {kw}")


@pytest.mark.parametrize("cfg", ["afiro", "support", "lazy500"])
def test_pageable_host_buffers_match_pinned(cfg, monkeypatch):
    """Pageable numpy buffers go through the pinned staging ring (parallel memcpy,
    several sub-batches in flight); results are bit-identical to the pinned path."""
    import ctypes
    from paper_1802_08557_b200 import _native, workloads
    if cfg == "afiro":
        A, b, c = workloads.afiro_arrays(30_000, seed=4)
        shared = False
    elif cfg == "support":
        A, b = workloads.support_polytope()
        c = workloads.support_directions(50_000)
        shared = True
    else:
        A, b, c = workloads.random_arrays(500, 40, seed=41)
        shared = False
    monkeypatch.setenv("BLP_STAGE_MB", "8")          # many sub-batches through a 4-slot ring
    lim = _native.make_limits()
    got = _native.solve_host(np.ascontiguousarray(A), np.ascontiguousarray(b), np.ascontiguousarray(c), lim,
                             shared_Ab=shared, out={k: np.zeros_like(v) for k, v in
                                                    _native.alloc_outputs(len(c), c.shape[1]).items()})
    pin = {k: _native.alloc_host(v.shape, v.dtype) for k, v in (("A", A), ("b", b), ("c", c))}
    for k, v in (("A", A), ("b", b), ("c", c)):
        pin[k][...] = v
    ref = _native.solve_host(pin["A"], pin["b"], pin["c"], lim, shared_Ab=shared)
    for k in ("status", "objective", "x", "it1", "it2"):
        assert np.array_equal(got[k], ref[k], equal_nan=True), k


def test_random_shapes_default_dispatch():
    """Thirty random (m, n) shapes through the default dispatcher (every family, the
    lazy-first path included), single- and two-phase LPs mixed: equal to the oracle."""
    from oracle import oracle
    from paper_1802_08557_b200 import batch_solve_arrays, workloads
    rng = np.random.default_rng(2026)
    for _ in range(30):
        m, n = int(rng.integers(1, 161)), int(rng.integers(1, 161))
        A1, b1, c1 = workloads.afiro_arrays(12, seed=int(rng.integers(1 << 30)), m=max(m, 2), n=n)
        A1, b1 = A1[:, :m], b1[:, :m]
        A2, b2, c2 = workloads.random_arrays(max(m, n), 12, seed=int(rng.integers(1 << 30)))
        A2, b2, c2 = A2[:, :m, :n], b2[:, :m], c2[:, :n]
        A = np.ascontiguousarray(np.concatenate([A1, A2]))
        b = np.ascontiguousarray(np.concatenate([b1, b2]))
        c = np.ascontiguousarray(np.concatenate([c1, c2]))
        want = oracle.solve_batch(A, b, c)
        compare(_native_dict(batch_solve_arrays(A, b, c)), want, f"random shape {m}x{n}")


def test_results_invariant_to_chunking_and_sharding(monkeypatch):
    """The reference's determinism law (test_acceptance.py:178-195) for every path:
    sub-batch counts, staging slot sizes, the object API's chunk plan and a two-shard
    run (devices=(0, 0)) all give bit-identical outcomes -- dense, lazy and deferred LPs."""
    from paper_1802_08557_b200 import BatchConfig, batch_solve, batch_solve_arrays, standard_form, workloads
    A1, b1, c1 = workloads.afiro_arrays(3000, seed=91, m=60, n=40)        # two-phase: deferred to pairlp
    A2, b2, c2 = workloads.random_arrays(60, 3000, seed=92)                 # single phase: lazy
    A = np.concatenate([A1, A2[:, :, :40]])
    b = np.concatenate([b1, b2])
    c = np.concatenate([c1, c2[:, :40]])
    ref = _native_dict(batch_solve_arrays(A, b, c))
    variants = [dict(BLP_HOST_CHUNKS="3"), dict(BLP_HOST_CHUNKS="64"), dict(BLP_HOST_TAPER="0"),
                dict(BLP_HOST_CHUNKS="5", BLP_HOST_TAPER="6"), dict(BLP_HOST_RAMP="0"), dict(BLP_HOST_RAMP="6"),
                dict(BLP_STAGE_MB="1"), dict(BLP_STAGE="0")]
    for env in variants:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        got = _native_dict(batch_solve_arrays(A, b, c))
        for k in ref:
            assert np.array_equal(ref[k], got[k], equal_nan=True), (env, k)
        for k in env:
            monkeypatch.delenv(k)
    got = _native_dict(batch_solve_arrays(A, b, c, devices=(0, 0)))
    for k in ref:
        assert np.array_equal(ref[k], got[k], equal_nan=True), ("sharded", k)
    lps = [standard_form(c[i], A[i], b[i]) for i in range(0, len(c), 7)]
    r1 = batch_solve(lps)
    r2 = batch_solve(lps, BatchConfig(memory_budget_bytes=lp_bytes_for(60, 40) * 37))
    assert r2.plan.count > 1
    for o1, o2 in zip(r1.outcomes, r2.outcomes):
        assert o1.status == o2.status and o1.iterations_phase1 == o2.iterations_phase1
        assert o1.iterations_phase2 == o2.iterations_phase2
        assert (o1.primal_point is None) == (o2.primal_point is None)
        if o1.primal_point is not None:
            assert np.array_equal(o1.primal_point, o2.primal_point) and o1.objective_value == o2.objective_value


def lp_bytes_for(m, n):
    from paper_1802_08557_b200 import lp_memory_bytes
    return lp_memory_bytes(m, n, num_slack=m, num_artificial=m)


@pytest.mark.parametrize("shape,shared", [((150, 150), False), ((64, 32), True), ((100, 100), False)])
def test_device_api_equals_host_api_lazy_paths(shape, shared):
    """The device entry point (torch tensors, caller's stream) takes the same lazy-first
    dispatch as the host one: identical results, independent and support mode."""
    from paper_1802_08557_b200 import SolverLimits, _native, workloads
    m, n = shape
    if shared:
        A, b = workloads.support_polytope()
        c = workloads.support_directions(5000)
    else:
        A1, b1, c1 = workloads.random_arrays(max(m, n), 200, seed=m + n)
        A2, b2, c2 = workloads.afiro_arrays(50, seed=m * n, m=m, n=n)
        A = np.concatenate([A1[:, :m, :n], A2])
        b = np.concatenate([b1[:, :m], b2])
        c = np.concatenate([c1[:, :n], c2])
    A, b, c = (np.ascontiguousarray(v) for v in (A, b, c))
    host = _native.solve_host(A, b, c, SolverLimits().to_native(), shared_Ab=shared)
    dev = torch.device("cuda:0")
    tA, tb, tc = (torch.from_numpy(v).to(dev) for v in (A, b, c))
    cnt = len(c)
    out = dict(status=torch.empty(cnt, dtype=torch.int8, device=dev),
               objective=torch.empty(cnt, dtype=torch.float64, device=dev),
               x=torch.empty(cnt, n, dtype=torch.float64, device=dev),
               it1=torch.empty(cnt, dtype=torch.int32, device=dev),
               it2=torch.empty(cnt, dtype=torch.int32, device=dev))
    stream = torch.cuda.Stream()
    _native.solve_device(tA, tb, tc, SolverLimits().to_native(), out, shared_Ab=shared, stream=stream)
    stream.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items()}
    for k in ("status", "objective", "x", "it1", "it2"):
        assert np.array_equal(got[k], host[k], equal_nan=True), (shape, k)
