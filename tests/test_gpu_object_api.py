"""The reference-facing object API (batch_solve(list[StandardFormLP]) -> BatchReport,
/root/reference/pkg/src/batchlp/batch.py:134-179) through the pointer-gather path
(_pyobj.collect + blp_solve_batch_gather) and the lazy OutcomeList: same outcomes as the
packed path, every kind of LP array the reference accepts, its errors in index order.
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


def _arrays_of(rep):
    outs = list(rep.outcomes)
    n = next((len(o.primal_point) for o in outs if o.primal_point is not None), 0)
    codes = {"optimal": 0, "unbounded": 1, "infeasible": 2, "iteration_limit": 3}
    return dict(status=np.array([codes[o.status.value] for o in outs]),
                objective=np.array([np.nan if o.objective_value is None else o.objective_value for o in outs]),
                x=np.array([o.primal_point if o.primal_point is not None else np.zeros(n) for o in outs]),
                it1=np.array([o.iterations_phase1 for o in outs]), it2=np.array([o.iterations_phase2 for o in outs]))


def test_object_api_equals_packed_and_oracle():
    from oracle import oracle
    from paper_1802_08557_b200 import BatchConfig, StandardFormLP, batch_solve, batch_solve_arrays, workloads
    A, b, c = workloads.afiro_arrays(30_000, seed=123)
    lps = [StandardFormLP(c=c[k], A=A[k], b=b[k]) for k in range(len(c))]
    rep = batch_solve(lps, BatchConfig(memory_budget_bytes=22_320 * 7_000))   # several planned chunks
    assert rep.plan.count >= 4 and len(rep.chunk_seconds) == rep.plan.count and len(rep.outcomes) == 30_000
    got = _arrays_of(rep)
    compare(got, oracle.solve_batch(A, b, c), "object api vs oracle")
    packed = batch_solve_arrays(A, b, c)
    assert rep.status_counts() == packed.status_counts()
    assert list(rep.status_counts()) == list(dict.fromkeys(o.status.value for o in rep.outcomes))   # first-occurrence order


def test_outcome_list_behaves_like_a_list():
    from paper_1802_08557_b200 import Status, batch_solve, gen_random_lps, solve
    lps = gen_random_lps(5, 50, seed=3)
    rep = batch_solve(lps)
    outs = rep.outcomes
    assert len(outs) == 50 and outs[0] is outs[0] and outs[-1] is outs[49]
    assert outs[10:13] == [outs[10], outs[11], outs[12]]
    for o, d in zip(outs, [solve(lp) for lp in lps]):
        assert (o.status, o.objective_value, o.iterations_phase1, o.iterations_phase2) == \
            (d.status, d.objective_value, d.iterations_phase1, d.iterations_phase2)
        assert np.array_equal(o.primal_point, d.primal_point)
    assert outs == outs[:]            # list equality (same SolveOutcome objects)
    with pytest.raises(IndexError):
        outs[50]
    assert all(o.status is Status.OPTIMAL for o in outs)


def test_slow_lps_are_coerced():
    """Lists, int arrays, Fortran-order and strided arrays, float32: coerced, same answers."""
    from paper_1802_08557_b200 import StandardFormLP, batch_solve, standard_form, workloads
    A, b, c = workloads.afiro_arrays(40, seed=9)
    lps = [standard_form(c[k], A[k], b[k]) for k in range(40)]
    want = _arrays_of(batch_solve(lps))
    odd = list(lps)
    odd[1] = StandardFormLP(c=list(c[1]), A=A[1].tolist(), b=list(b[1]))
    odd[2] = StandardFormLP(c=c[2].astype(np.int64), A=A[2].astype(np.int64), b=b[2].astype(np.int64))
    odd[3] = StandardFormLP(c=c[3], A=np.asfortranarray(A[3]), b=b[3])
    big = np.zeros((28, 64))
    big[:, ::2] = A[4]
    odd[4] = StandardFormLP(c=c[4], A=big[:, ::2], b=b[4])
    odd[5] = StandardFormLP(c=c[5].astype(np.float32), A=A[5], b=b[5])
    got = _arrays_of(batch_solve(odd))
    for key in ("status", "it1", "it2", "x"):
        assert np.array_equal(got[key], want[key]), key


def test_errors_in_index_order():
    from paper_1802_08557_b200 import HeterogeneousBatch, StandardFormLP, batch_solve, standard_form
    ok = standard_form([1.0, 2.0], [[1.0, 1.0]], [4.0])
    with pytest.raises(HeterogeneousBatch):
        batch_solve([ok, standard_form([1.0], [[1.0]], [1.0])])
    ragged = StandardFormLP(c=np.array([1.0, 2.0]), A=[[1.0, 1.0, 3.0]], b=np.array([4.0]))
    with pytest.raises(ValueError, match="row 0 has 3 coefficients, expected 2"):
        batch_solve([ok, ragged, ok])
    nan_first = standard_form([1.0, 2.0], [[np.nan, 1.0]], [4.0])
    with pytest.raises(ValueError, match=r"A\[0\]\[0\] is not finite"):
        batch_solve([ok, nan_first, ragged])
    text = StandardFormLP(c=np.array([1.0, 2.0]), A=[["x", 1.0]], b=np.array([4.0]))
    with pytest.raises(ValueError, match="row 0 is not numeric"):
        batch_solve([ok, text])


def test_object_api_on_lazy_and_support_shapes():
    """Shapes outside the condensed family (lazy + dense fallbacks) and a shared polytope."""
    from oracle import oracle
    from paper_1802_08557_b200 import StandardFormLP, batch_solve, workloads
    A, b, c = workloads.random_arrays(150, 30, seed=4)
    rep = batch_solve([StandardFormLP(c=c[k], A=A[k], b=b[k]) for k in range(30)])
    compare(_arrays_of(rep), oracle.solve_batch(A, b, c), "object api 150x150")
    P, q = workloads.support_polytope()
    C = workloads.support_directions(3000)
    rep = batch_solve([StandardFormLP(c=C[k], A=P, b=q) for k in range(3000)])
    compare(_arrays_of(rep), oracle.solve_batch(P, q, C, shared_Ab=True), "object api support")


def test_two_rank_bench_on_one_gpu():
    """bench.py's multi-rank path (one process per rank, torchrun) with both ranks folded onto
    the one visible GPU (BLP_BENCH_SHARE_GPU=1: gloo for the scalar collectives): the line
    reports the whole job, and each rank's timed outputs match the oracle on its shard."""
    import json
    import os
    import socket
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, BLP_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(root / "bench.py"), "--gpus", "2",
           "--count", "20000", "--steps", "3", "--warmup", "3"]
    p = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 40_000 and d["config"]["lps_per_gpu"] == 20_000
    pr = d["parity"]
    assert pr["checked"] == 10_000 and pr["of"] == 40_000
    assert pr["status_mismatch"] == pr["x_mismatch"] == pr["iter_mismatch"] == 0 and pr["max_obj_rel"] <= 1e-9
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] >= 3


def test_object_api_shared_polytope_is_support_mode(monkeypatch):
    """LPs of a list that all point at one A and one b (the support-function workload through
    the reference API) are solved in support mode -- phase 1 shared -- with outputs equal to
    the oracle's per-LP solves and to the library's per-LP path (BLP_GATHER_SHARED=0);
    equal-valued but distinct arrays take the per-LP path."""
    from oracle import oracle
    from paper_1802_08557_b200 import StandardFormLP, batch_solve, workloads
    A, b = workloads.support_polytope_two_phase()
    C = workloads.support_directions(4000, offset=9)
    lps = [StandardFormLP(c=C[k], A=A, b=b) for k in range(len(C))]
    want = oracle.solve_batch(A, b, C, shared_Ab=True, threads=oracle.host_cores())
    compare(_arrays_of(batch_solve(lps)), want, "object api shared two-phase polytope")
    monkeypatch.setenv("BLP_GATHER_SHARED", "0")
    compare(_arrays_of(batch_solve(lps)), want, "object api shared polytope, per-LP path")
    monkeypatch.delenv("BLP_GATHER_SHARED")
    lps2 = [StandardFormLP(c=C[k], A=A.copy(), b=b.copy()) for k in range(300)]
    compare(_arrays_of(batch_solve(lps2)), {k: v[:300] for k, v in want.items() if k != "threads"},
            "object api distinct copies")
