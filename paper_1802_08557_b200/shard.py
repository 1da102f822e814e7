"""LP-index sharding across GPUs / ranks.

LPs are independent, so a batch splits into contiguous index ranges with no
collective on the data path: each device solves its range and the results
land in the matching slices of the caller's output arrays (host-side gather).
The same rule serves the multi-device host API (``batch._solve_sharded``) and
the multi-rank benchmark (one process per GPU).
"""
from __future__ import annotations


def shard_bounds(count: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous [start, end) ranges covering [0, count) in order, sizes differing by at most one.

    Empty ranges are dropped, so fewer than ``parts`` ranges come back when count < parts.
    """
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if count < 0:
        raise ValueError("count must be >= 0")
    base, extra = divmod(count, parts)
    out, start = [], 0
    for k in range(parts):
        size = base + (1 if k < extra else 0)
        if size:
            out.append((start, start + size))
        start += size
    return out


def rank_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """This rank's [start, end) of a count-LP global batch (may be empty)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(count, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)
