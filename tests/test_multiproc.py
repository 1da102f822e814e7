"""Multi-rank / multi-device sharding on CPU: the product's own sharding and gather code
(paper_1802_08557_b200.multirank, batch._solve_sharded) with an injected per-device solver,
since there is no GPU here (the GPU path itself is covered by the -m gpu tests, including a
two-rank bench run).

The batch shards with no collective on the data path: each rank solves a
contiguous LP-index range and rank 0 gathers results into index order; bench.py's only
other collectives are a barrier and MAX/SUM reductions of scalars, exercised here too.
The injected solver is the CPU oracle (the parity checker) -- test-only.
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_08557_b200.shard import rank_range, shard_bounds


def test_shard_bounds_cover_in_order():
    for count in (0, 1, 7, 100, 100_001):
        for parts in (1, 2, 3, 8):
            b = shard_bounds(count, parts)
            assert [i for s, e in b for i in range(s, e)] == list(range(count))
            sizes = [e - s for s, e in b]
            assert not sizes or max(sizes) - min(sizes) <= 1
            ranges = [rank_range(count, r, parts) for r in range(parts)]
            assert [r for r in ranges if r[1] > r[0]] == b
    with pytest.raises(ValueError):
        shard_bounds(5, 0)


def _oracle_solver(A, b, c, shared_Ab, device, limits):
    from oracle import oracle
    r = oracle.solve_batch(A, b, c, shared_Ab=shared_Ab, threads=1, max_iterations=limits.max_iterations,
                           anti_cycling=limits.anti_cycling, degenerate_pivot_limit=limits.degenerate_pivot_limit)
    return {k: r[k] for k in ("status", "objective", "x", "it1", "it2")}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, A, b, c, shared, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1802_08557_b200 import multirank
    s, e, res = multirank.solve_shard(A, b, c, rank, world, shared_Ab=shared, device=rank, solver=_oracle_solver)
    whole = multirank.gather_shards(s, e, res, len(c))
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)     # bench.py's max-over-ranks timing
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out_q.put((whole, float(t.item())))
    else:
        assert whole is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shared", [False, True])
def test_two_rank_shards_gather_to_single_process(shared):
    from oracle import oracle
    from paper_1802_08557_b200 import workloads
    if shared:
        A, b = workloads.support_polytope()
        c = workloads.support_directions(301)
    else:
        A, b, c = workloads.afiro_arrays(301, seed=31)
    want = oracle.solve_batch(A, b, c, shared_Ab=shared, threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, A, b, c, shared, q)) for r in range(2)]
    for p in procs:
        p.start()
    whole, tmax = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    for k in ("status", "x", "it1", "it2"):
        assert np.array_equal(whole[k], want[k]), k
    opt = want["status"] == 0
    assert np.array_equal(whole["objective"][opt], want["objective"][opt])


def test_multi_device_host_api_shards_and_gathers():
    """batch._solve_sharded over four 'devices' (one host thread each) writes every shard into
    its slice of one output set: equal to the unsharded solve, also for fewer LPs than devices."""
    from paper_1802_08557_b200 import SolverLimits, workloads
    from paper_1802_08557_b200.batch import _solve_sharded
    seen = []
    lock = threading.Lock()

    def fake_native(A, b, c, lim, *, shared_Ab, device, out):
        from oracle import oracle
        with lock:
            seen.append((device, len(c)))
        r = oracle.solve_batch(A, b, c, shared_Ab=shared_Ab, threads=1)
        for k in ("status", "objective", "x", "it1", "it2"):
            out[k][...] = r[k]
        return out

    def outputs(count, n):
        return dict(status=np.empty(count, np.int8), objective=np.empty(count), x=np.empty((count, n)),
                    it1=np.empty(count, np.int32), it2=np.empty(count, np.int32))

    from oracle import oracle
    A, b, c = workloads.afiro_arrays(403, seed=5)
    want = oracle.solve_batch(A, b, c, threads=1)
    got = _solve_sharded(A, b, c, SolverLimits(), (0, 1, 2, 3), False, out=outputs(403, 32), solve_host=fake_native)
    assert sorted(seen) == [(0, 101), (1, 101), (2, 101), (3, 100)]
    for k in ("status", "x", "it1", "it2"):
        assert np.array_equal(got[k], want[k]), k
    seen.clear()
    got = _solve_sharded(A[:2], b[:2], c[:2], SolverLimits(), (0, 1, 2, 3), False, out=outputs(2, 32),
                         solve_host=fake_native)
    assert sorted(seen) == [(0, 1), (1, 1)]
    assert np.array_equal(got["x"], want["x"][:2])
