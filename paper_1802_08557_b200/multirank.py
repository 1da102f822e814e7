"""One process per GPU (torch.distributed): LP-index shards and the host-side gather.

The batch shards with no collective on the data path (the
reference's only parallel path is its process pool, batch.py:160-171): rank r
solves the contiguous range ``rank_range(count, r, world)`` on its own GPU, and
the only communication is the result gather to rank 0 (or nothing at all, when
every rank keeps its shard).  ``solve_shard`` / ``gather_shards`` are what
bench.py's multi-rank path runs; the per-rank solver is injectable so the
sharding and gather logic is testable on CPU ranks (gloo) where no GPU exists.
"""
from __future__ import annotations

from typing import Callable

import numpy as np

from .shard import rank_range

RESULT_KEYS = ("status", "objective", "x", "it1", "it2")


def solve_shard(A, b, c, rank: int, world: int, *, shared_Ab: bool = False, device: int = 0, limits=None,
                solver: Callable | None = None) -> tuple[int, int, dict]:
    """Solve this rank's contiguous slice of a packed global batch on `device`.

    Returns (start, end, result dict with RESULT_KEYS).  `solver(A, b, c, shared_Ab, device, limits)`
    defaults to the GPU library (batch_solve_arrays / support_batch)."""
    from .simplex import SolverLimits
    limits = limits or SolverLimits()
    s, e = rank_range(len(c), rank, world)
    As, bs = (A, b) if shared_Ab else (A[s:e], b[s:e])
    if solver is None:
        solver = _gpu_solver
    return s, e, solver(As, bs, c[s:e], shared_Ab, device, limits)


def _gpu_solver(A, b, c, shared_Ab: bool, device: int, limits) -> dict:
    from .batch import batch_solve_arrays, support_batch
    if len(c) == 0:
        n = c.shape[1]
        return dict(status=np.empty(0, np.int8), objective=np.empty(0), x=np.empty((0, n)),
                    it1=np.empty(0, np.int32), it2=np.empty(0, np.int32))
    r = (support_batch if shared_Ab else batch_solve_arrays)(A, b, c, limits, devices=(device,))
    return dict(status=r.status, objective=r.objective, x=r.x, it1=r.iterations_phase1, it2=r.iterations_phase2)


def gather_shards(start: int, end: int, res: dict, count: int, *, group=None, dst: int = 0) -> dict | None:
    """Host-side gather of every rank's (start, end, result) into index order on rank `dst`
    (None elsewhere).  One gather_object per call: results are small (x is count x n)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    payload = (start, end, {k: np.asarray(res[k]) for k in RESULT_KEYS})
    parts = [None] * world if rank == dst else None
    dist.gather_object(payload, parts, dst=dst, group=group)
    if rank != dst:
        return None
    n = next((p[2]["x"].shape[1] for p in parts if p[2]["x"].ndim == 2), 0)
    out = dict(status=np.empty(count, np.int8), objective=np.empty(count), x=np.empty((count, n)),
               it1=np.empty(count, np.int32), it2=np.empty(count, np.int32))
    covered = 0
    for s, e, r in sorted(parts, key=lambda p: p[0]):
        if s != covered:
            raise RuntimeError(f"shards do not tile the batch: gap at {covered}, next shard starts at {s}")
        for k in RESULT_KEYS:
            out[k][s:e] = r[k]
        covered = e
    if covered != count:
        raise RuntimeError(f"shards cover {covered} of {count} LPs")
    return out
