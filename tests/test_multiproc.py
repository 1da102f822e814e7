"""Multi-rank sharding on CPU (gloo, world_size 2): the LP-index split and the host-side
gather reproduce the single-process result, and max-over-ranks timing is what rank 0 sees.

The batch shards with no collective on the data path; the only
collectives bench.py uses are a barrier and a MAX/SUM reduction of scalars, which
is what is exercised here.  The per-rank "solver" is the CPU oracle on the rank's
slice (the GPU solve is covered by the -m gpu parity tests).
"""
import os
import socket

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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, A, b, c, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    s, e = rank_range(len(c), rank, world)
    res = oracle.solve_batch(A[s:e], b[s:e], c[s:e], threads=1)
    # host-side gather of the shards (what the multi-device API does with slices)
    parts = [None] * world
    dist.all_gather_object(parts, (s, e, res["status"], res["x"], res["it1"], res["it2"]))
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out_q.put((parts, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_process():
    from oracle import oracle
    from paper_1802_08557_b200 import workloads
    A, b, c = workloads.afiro_arrays(300, seed=31)
    whole = oracle.solve_batch(A, b, c, threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, A, b, c, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    status = np.concatenate([p[2] for p in sorted(parts)])
    x = np.concatenate([p[3] for p in sorted(parts)])
    it = np.concatenate([p[4] + p[5] for p in sorted(parts)])
    assert [p[0] for p in sorted(parts)] == [0, 150]
    assert np.array_equal(status, whole["status"]) and np.array_equal(x, whole["x"])
    assert np.array_equal(it, whole["it1"] + whole["it2"])
