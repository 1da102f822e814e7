"""Batched hyper-rectangle LPs on the GPU (the paper's Eq. 7 kernel).

Mirrors /root/reference/pkg/src/batchlp/boxlp.py: ``BoxLP`` (:20-34),
``BoxSolution`` (:37-40), ``InvalidBox`` (:16-17), ``solve_box`` (:44-55)
and ``solve_box_batch`` (:72-83) -- same results, the same InvalidBox
messages, invalid boxes recorded in place -- with the arithmetic in
blp_box_kernel.cuh.  ``box_batch_arrays`` is the packed path (lower, upper,
direction as [count, n] arrays).  Values agree with the reference to 1e-9
(it sums direction @ point with BLAS ddot); points are exact.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native


class InvalidBox(Exception):
    """Some lower bound exceeds its upper bound, or a bound is not finite."""


@dataclass(frozen=True)
class BoxLP:
    lower: np.ndarray
    upper: np.ndarray
    direction: np.ndarray

    @property
    def n(self) -> int:
        return len(self.direction)

    @classmethod
    def build(cls, lower, upper, direction) -> "BoxLP":
        return cls(np.asarray(lower, dtype=float), np.asarray(upper, dtype=float),
                   np.asarray(direction, dtype=float))


@dataclass(frozen=True)
class BoxSolution:
    value: float
    point: np.ndarray


@dataclass
class BoxArrays:
    """Packed results: value (NaN if invalid), point [count, n], status (0 ok, -1 non-finite
    bound, k+1 lower[k] > upper[k])."""

    value: np.ndarray
    point: np.ndarray
    status: np.ndarray


def _invalid(status: int, lower: np.ndarray, upper: np.ndarray) -> InvalidBox:
    if status < 0:
        return InvalidBox("box bounds must be finite")
    j = status - 1
    return InvalidBox(f"lower[{j}] = {lower[j]} > upper[{j}] = {upper[j]}")


def box_batch_arrays(lower, upper, direction, *, device: int = 0) -> BoxArrays:
    lower = np.ascontiguousarray(lower, dtype=np.float64)
    upper = np.ascontiguousarray(upper, dtype=np.float64)
    direction = np.ascontiguousarray(direction, dtype=np.float64)
    if not (lower.shape == upper.shape == direction.shape and direction.ndim == 2):
        raise ValueError(f"box arrays disagree: {lower.shape}, {upper.shape}, {direction.shape}")
    res = _native.box_solve_host(lower, upper, direction, device=device)
    return BoxArrays(res["value"], res["point"], res["status"])


def solve_box(box: BoxLP) -> BoxSolution:
    """Maximise direction.x over the box (boxlp.py:44-55); raises InvalidBox."""
    res = box_batch_arrays(np.asarray(box.lower, float)[None], np.asarray(box.upper, float)[None],
                           np.asarray(box.direction, float)[None])
    if res.status[0] != 0:
        raise _invalid(int(res.status[0]), np.asarray(box.lower, float), np.asarray(box.upper, float))
    return BoxSolution(value=float(res.value[0]), point=np.array(res.point[0]))


def solve_box_batch(boxes: Sequence[BoxLP], workers: int = 1) -> list[BoxSolution | InvalidBox]:
    """Element-wise solve_box over a batch (boxlp.py:72-83): order preserved, invalid boxes
    recorded in place as the InvalidBox instance.  Same-dimension boxes are packed into one
    launch per dimension; ``workers`` is accepted for compatibility only."""
    boxes = list(boxes)
    out: list[BoxSolution | InvalidBox | None] = [None] * len(boxes)
    by_dim: dict[int, list[int]] = {}
    for k, b in enumerate(boxes):
        by_dim.setdefault(len(b.direction), []).append(k)
    for n, idx in by_dim.items():
        lo = np.array([np.asarray(boxes[k].lower, float) for k in idx]).reshape(len(idx), n)
        hi = np.array([np.asarray(boxes[k].upper, float) for k in idx]).reshape(len(idx), n)
        d = np.array([np.asarray(boxes[k].direction, float) for k in idx]).reshape(len(idx), n)
        res = box_batch_arrays(lo, hi, d)
        for r, k in enumerate(idx):
            st = int(res.status[r])
            out[k] = BoxSolution(float(res.value[r]), np.array(res.point[r])) if st == 0 else \
                _invalid(st, lo[r], hi[r])
    return out
