"""Host-side logic of the drop-in, no GPU needed: the reference's batch/model/simplex API
contracts (restating /root/reference/pkg/tests/test_batch.py, test_model.py) and the
loud failure of the product path without CUDA."""
import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1802_08557_b200 import (
    BatchConfig,
    BatchTooLarge,
    HeterogeneousBatch,
    NativeUnavailable,
    SolverLimits,
    StandardFormLP,
    Status,
    batch_solve,
    gen_random_lps,
    lp_memory_bytes,
    plan_chunks,
    standard_form,
    validate,
    workloads,
)


class TestMemoryModel:                      # test_batch.py:18-31
    def test_reference_shape(self):
        assert lp_memory_bytes(m=5, n=5, num_slack=5, num_artificial=0) == 768

    def test_degenerate_dimensions(self):
        assert lp_memory_bytes(m=0, n=0, num_slack=0, num_artificial=0) == 48

    def test_linear_in_data_size(self):
        assert lp_memory_bytes(7, 3, 7, 2, 8) == 2 * lp_memory_bytes(7, 3, 7, 2, 4)

    def test_formula(self):                 # test_acceptance.py:127-141
        rng = np.random.default_rng(202405)
        for _ in range(20):
            m, n, slack, arti = (int(v) for v in rng.integers(0, 200, 4))
            ds = int(rng.choice([4, 8]))
            cols = n + slack + arti + 2
            assert lp_memory_bytes(m, n, slack, arti, ds) == (m + 1) * cols * ds + 2 * cols * ds


class TestPlanChunks:                       # test_batch.py:34-70
    def test_worked_example(self):
        plan = plan_chunks(3000, 768, BatchConfig(memory_budget_bytes=1_000_000))
        assert plan.batch_size == 1302
        assert plan.sizes == (1302, 1302, 396)
        assert plan.bounds == ((0, 1302), (1302, 2604), (2604, 3000))

    def test_empty(self):
        assert plan_chunks(0, 10, BatchConfig()).bounds == ()

    def test_single_chunk(self):
        assert plan_chunks(5, 10, BatchConfig(memory_budget_bytes=1000)).bounds == ((0, 5),)

    def test_single_lp_over_budget(self):
        with pytest.raises(BatchTooLarge):
            plan_chunks(1, 2000, BatchConfig(memory_budget_bytes=1000))

    @settings(max_examples=200)
    @given(st.integers(0, 5000), st.integers(1, 4000), st.integers(1, 10_000_000))
    def test_exact_cover(self, count, lp_bytes, budget):
        if lp_bytes > budget:
            with pytest.raises(BatchTooLarge):
                plan_chunks(count, lp_bytes, BatchConfig(memory_budget_bytes=budget))
            return
        plan = plan_chunks(count, lp_bytes, BatchConfig(memory_budget_bytes=budget))
        assert plan.batch_size == budget // lp_bytes or count == 0
        flat = [i for s, e in plan.bounds for i in range(s, e)]
        assert flat == list(range(count))
        assert all(e > s for s, e in plan.bounds)
        if count:
            assert plan.count == math.ceil(count / plan.batch_size)


class TestConfig:
    def test_invariants(self):
        with pytest.raises(ValueError):
            BatchConfig(memory_budget_bytes=0)
        with pytest.raises(ValueError):
            BatchConfig(worker_count=0)
        with pytest.raises(ValueError):
            BatchConfig(devices=())

    def test_limits(self):                  # simplex.py:34-60
        with pytest.raises(ValueError):
            SolverLimits(max_iterations=0)
        assert SolverLimits().iterations_for(28, 32) == 50 * 60
        assert SolverLimits(max_iterations=7).iterations_for(28, 32) == 7
        assert SolverLimits().bland_trigger(0) == 1
        assert SolverLimits(degenerate_pivot_limit=0).bland_trigger(5) == 0
        lim = SolverLimits(max_iterations=3, anti_cycling=False, degenerate_pivot_limit=2).to_native()
        assert (lim.max_iterations, lim.anti_cycling, lim.degenerate_limit) == (3, 0, 2)
        d = SolverLimits().to_native()
        assert (d.max_iterations, d.anti_cycling, d.degenerate_limit) == (0, 1, -1)


class TestBatchSolveHost:
    def test_empty_batch(self):
        report = batch_solve([])
        assert report.outcomes == [] and report.plan.bounds == () and report.chunk_seconds == []

    def test_heterogeneous_shapes_rejected_before_any_gpu_work(self):
        lps = [gen_random_lps(3, 1, seed=0)[0], gen_random_lps(4, 1, seed=0)[0]]
        with pytest.raises(HeterogeneousBatch, match=r"batch mixes LP shapes \[\(3, 3\), \(4, 4\)\]"):
            batch_solve(lps)

    def test_budget_accounts_for_artificials(self):
        lps = gen_random_lps(3, 4, seed=10, feasible_start=False)
        with pytest.raises(BatchTooLarge):
            batch_solve(lps, BatchConfig(memory_budget_bytes=lp_memory_bytes(3, 3, 3, 0)))

    def test_no_cpu_fallback(self, monkeypatch):
        """Without a visible GPU the product path raises instead of computing on the host."""
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
        with pytest.raises(NativeUnavailable):
            batch_solve(gen_random_lps(3, 2, seed=1))


class TestModel:                            # model.py:263-301 messages
    def test_validate_messages(self):
        assert validate(standard_form([1.0], [[1.0]], [1.0])) == []
        assert validate(standard_form([np.nan], [[1.0]], [1.0])) == ["c[0] is not finite"]
        assert validate(standard_form([1.0], [[np.inf]], [1.0])) == ["A[0][0] is not finite"]
        assert validate(standard_form([1.0], [[1.0]], [np.nan])) == ["b[0] is not finite"]
        bad = StandardFormLP(c=np.ones(2), A=np.ones((1, 3)), b=np.ones(1))
        assert validate(bad) == ["row 0 has 3 coefficients, expected 2"]
        assert validate(StandardFormLP(c=np.ones(2), A=np.ones((2, 2)), b=np.ones(1))) == \
            ["A has 2 rows, expected 1"]

    def test_validate_matches_reference(self, reference):
        cases = [([1.0, np.nan], [[1.0, 2.0]], [1.0]), ([1.0], [[np.inf], [1.0]], [np.nan, 2.0]),
                 ([1.0, 2.0], [[1.0, 2.0]], [3.0])]
        for c, A, b in cases:
            mine = validate(standard_form(c, A, b))
            ref = reference.validate(reference.standard_form(c, A, b))
            assert mine == ref

    def test_status_values(self):
        assert [s.value for s in Status] == ["optimal", "unbounded", "infeasible", "iteration_limit"]


class TestWorkloads:
    def test_gen_random_lps_matches_reference(self, reference):
        for dim, count, seed, fs in ((5, 20, 0, True), (3, 7, 10, False), (50, 2, 5, True)):
            mine = gen_random_lps(dim, count, seed, fs)
            ref = reference.gen_random_lps(dim, count, seed, fs)
            for a, r in zip(mine, ref):
                assert np.array_equal(a.A, r.A) and np.array_equal(a.b, r.b) and np.array_equal(a.c, r.c)

    def test_recipes_are_deterministic_and_shaped(self):
        A, b, c = workloads.afiro_arrays(50)
        A2, b2, c2 = workloads.afiro_arrays(50)
        assert A.shape == (50, 28, 32) and b.shape == (50, 28) and c.shape == (50, 32)
        assert np.array_equal(A, A2) and np.array_equal(b, b2) and np.array_equal(c, c2)
        assert (b < 0).any(axis=1).mean() > 0.9       # two-phase: mixed-sign b
        A, b, c = workloads.degenerate_arrays(40)
        assert A.shape == (40, 100, 100)
        Ap, bp = workloads.support_polytope()
        assert Ap.shape == (64, 32) and (bp > 0).all()

    def test_padded_beale_embeds_beale(self):
        A, b, c = workloads.padded_beale(100, 100)
        assert np.array_equal(A[:3, :4], workloads.BEALE_A) and (b[3:] == 1).all() and (c[4:] == -1).all()
