"""Batched entry points of the drop-in.

``batch_solve(lps, config) -> BatchReport`` keeps the reference signature and
result layout (/root/reference/pkg/src/batchlp/batch.py:134-179): same-shape
check (``HeterogeneousBatch``, :141-144), the Algorithm-1 chunk plan computed
with the batch-worst artificial count (:146-153, ``lp_memory_bytes`` :98-106,
``plan_chunks`` :109-127, ``BatchTooLarge``), outcomes in input order, one
``chunk_seconds`` entry per planned chunk, ``total_seconds``.

What changes is underneath: the LPs are packed once into contiguous arrays
(one copy), validated inside the kernel's tableau build (non-finite entries), and
each planned chunk is one call into libblp.so, which pipelines sub-batches
over CUDA streams on the GPU(s).  ``worker_count`` stays what it is in the
reference -- a throughput knob that never changes results -- and is unused
by the GPU path; ``devices`` chooses the GPUs (contiguous LP-index shards,
no collective).

``batch_solve_arrays`` / ``support_batch`` are the packed fast paths that
skip the ``StandardFormLP`` / ``SolveOutcome`` object layers.
"""
from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass, field
from collections.abc import Sequence

import numpy as np

from . import _native
from .model import SolveOutcome, StandardFormLP, STATUS_BY_CODE, invalid_message, validate
from .shard import shard_bounds
from .simplex import PHASE1_UNBOUNDED_MESSAGE, SolverLimits, outcome_from_arrays, outcomes_from_arrays

# Column ceiling of the paper's one-block-per-LP Kepler kernel (batch.py:25-29);
# informational, as in the reference.  The B200 kernels have no such limit.
REFERENCE_GPU_BLOCK_COLS = 1024


class BatchTooLarge(Exception):
    """A single LP's tableau exceeds the memory budget."""


class HeterogeneousBatch(Exception):
    """The LPs in a batch do not all share one (m, n) shape."""


@dataclass(frozen=True)
class BatchConfig:
    """Knobs for one batched run (batch.py:40-58) plus the GPU selection.

    ``memory_budget_bytes`` governs the chunk plan only; ``worker_count`` is
    accepted for compatibility (results never depend on it); ``devices``
    lists the CUDA devices the batch is sharded over (default: device 0).
    """

    memory_budget_bytes: int = 1 << 30
    worker_count: int = 1
    limits: SolverLimits = field(default_factory=SolverLimits)
    data_size_bytes: int = 8
    devices: tuple[int, ...] = (0,)

    def __post_init__(self):
        if self.memory_budget_bytes <= 0:
            raise ValueError("memory_budget_bytes must be positive")
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")
        if len(self.devices) < 1:
            raise ValueError("devices must name at least one CUDA device")


@dataclass(frozen=True)
class ChunkPlan:
    """Contiguous [start, end) pieces covering the batch, in order (batch.py:61-74)."""

    batch_size: int
    bounds: tuple[tuple[int, int], ...]

    @property
    def sizes(self) -> tuple[int, ...]:
        return tuple(e - s for s, e in self.bounds)

    @property
    def count(self) -> int:
        return len(self.bounds)


@dataclass
class BatchReport:
    """Outcomes in input order plus plan and timings (batch.py:77-95)."""

    outcomes: Sequence[SolveOutcome]   # an OutcomeList (list-like, built on access) from batch_solve
    plan: ChunkPlan
    chunk_seconds: list[float]
    total_seconds: float

    @property
    def lps_per_second(self) -> float:
        if self.total_seconds <= 0:
            return float("inf")
        return len(self.outcomes) / self.total_seconds

    def status_counts(self) -> dict[str, int]:
        if isinstance(self.outcomes, OutcomeList):
            return self.outcomes.status_counts()
        counts: dict[str, int] = {}
        for o in self.outcomes:
            counts[o.status.value] = counts.get(o.status.value, 0) + 1
        return counts


def lp_memory_bytes(m: int, n: int, num_slack: int, num_artificial: int, data_size_bytes: int = 8) -> int:
    """Reference per-LP footprint (Eq. 5): tableau + two scan arrays (batch.py:98-106)."""
    cols = n + num_slack + num_artificial + 2
    return (m + 1 + 2) * cols * data_size_bytes


def plan_chunks(count: int, lp_bytes: int, config: BatchConfig) -> ChunkPlan:
    """Algorithm 1 (batch.py:109-127): chunks of floor(S / lp_bytes) LPs, last one the remainder."""
    if lp_bytes > config.memory_budget_bytes:
        raise BatchTooLarge(f"one LP needs {lp_bytes} bytes but the budget is {config.memory_budget_bytes}")
    if count == 0:
        return ChunkPlan(batch_size=0, bounds=())
    size = config.memory_budget_bytes // lp_bytes
    if count <= size:
        return ChunkPlan(batch_size=size, bounds=((0, count),))
    return ChunkPlan(batch_size=size, bounds=tuple(
        (k * size, min((k + 1) * size, count)) for k in range(math.ceil(count / size))))


# ---------------------------------------------------------------------------
# packed fast paths

@dataclass
class BatchArrays:
    """Packed results: status codes (include/blp.h), objective (NaN unless optimal),
    x [B, n] (zeros unless optimal), per-phase iteration counts."""

    status: np.ndarray
    objective: np.ndarray
    x: np.ndarray
    iterations_phase1: np.ndarray
    iterations_phase2: np.ndarray

    def outcome(self, k: int) -> SolveOutcome:
        return outcome_from_arrays(self._as_dict(), k)

    def outcomes(self) -> list[SolveOutcome]:
        d = self._as_dict()
        return outcomes_from_arrays(d, 0, len(self.status))

    def status_counts(self) -> dict[str, int]:
        codes, counts = np.unique(self.status, return_counts=True)
        return {STATUS_BY_CODE[c].value: int(k) for c, k in zip(codes, counts) if c < len(STATUS_BY_CODE)}

    def _as_dict(self) -> dict:
        return dict(status=self.status, objective=self.objective, x=self.x,
                    it1=self.iterations_phase1, it2=self.iterations_phase2)


def _as_f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _solve_sharded(A, b, c, limits: SolverLimits, devices: Sequence[int], shared_Ab: bool,
                   out: dict | None = None, solve_host=None) -> dict:
    """Contiguous LP-index shards, one host thread per device (ctypes releases the GIL); each
    shard's results land in its slice of `out` (the host-side gather).  `solve_host` is the
    per-device solver, _native.solve_host (the GPU library) unless a test injects one."""
    solve_host = solve_host or _native.solve_host
    count, n = c.shape
    if out is None:
        out = _native.alloc_outputs(count, n) if count else dict(
            status=np.empty(0, np.int8), objective=np.empty(0), x=np.empty((0, n)),
            it1=np.empty(0, np.int32), it2=np.empty(0, np.int32))
    lim = limits.to_native()
    devices = list(devices)[:max(1, count)]
    if len(devices) == 1 or count == 0:
        if count:
            solve_host(A, b, c, lim, shared_Ab=shared_Ab, device=devices[0], out=out)
        return out
    errors: list[BaseException] = []

    def work(dev: int, s: int, e: int) -> None:
        try:
            sub = {k: v[s:e] for k, v in out.items()}
            solve_host(A if shared_Ab else A[s:e], b if shared_Ab else b[s:e], c[s:e], lim,
                       shared_Ab=shared_Ab, device=dev, out=sub)
        except BaseException as err:  # re-raised on the caller's thread
            errors.append(err)

    threads = [threading.Thread(target=work, args=(d, s, e))
               for d, (s, e) in zip(devices, shard_bounds(count, len(devices)))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out


def batch_solve_arrays(A, b, c, limits: SolverLimits = SolverLimits(), *,
                       devices: Sequence[int] = (0,)) -> BatchArrays:
    """Solve a packed batch: A [B,m,n], b [B,m], c [B,n] (fp64).  GPU only.

    Finiteness is validated inside the kernel's tableau build; the first LP
    with a non-finite entry raises the reference's ValueError, an LP whose
    phase 1 reports unbounded raises RuntimeError (whichever comes first).
    """
    A, b, c = _as_f64(A), _as_f64(b), _as_f64(c)
    if A.ndim != 3 or b.ndim != 2 or c.ndim != 2 or A.shape != (c.shape[0], b.shape[1], c.shape[1]) \
            or b.shape[0] != c.shape[0]:
        raise ValueError(f"packed shapes disagree: A {A.shape}, b {b.shape}, c {c.shape}")
    res = _solve_sharded(A, b, c, limits, devices, shared_Ab=False)
    _raise_for_errors(res, lambda k: StandardFormLP(c=c[k], A=A[k], b=b[k]))
    return _arrays(res)


def support_batch(A, b, C, limits: SolverLimits = SolverLimits(), *, devices: Sequence[int] = (0,)) -> BatchArrays:
    """Support-function mode: one polytope A x <= b (A [m,n], b [m]) and many
    objective directions C [B,n]; LP k maximises C[k].x over the polytope.

    Same results as batch_solve over [StandardFormLP(C[k], A, b)],
    without replicating A per LP.
    """
    A, b, C = _as_f64(A), _as_f64(b), _as_f64(C)
    if A.ndim != 2 or b.ndim != 1 or C.ndim != 2 or A.shape != (b.shape[0], C.shape[1]):
        raise ValueError(f"support shapes disagree: A {A.shape}, b {b.shape}, C {C.shape}")
    res = _solve_sharded(A, b, C, limits, devices, shared_Ab=True)
    _raise_for_errors(res, lambda k: StandardFormLP(c=C[k], A=A, b=b))
    return _arrays(res)


def _raise_for_errors(res: dict, lp_of) -> None:
    """Reference error behaviour for the first failing LP in index order."""
    bad = np.flatnonzero(res["status"] >= 4)
    if bad.size:
        k = int(bad[0])
        if res["status"][k] == 5:
            raise ValueError(invalid_message(validate(lp_of(k))))
        raise RuntimeError(PHASE1_UNBOUNDED_MESSAGE)


def _arrays(res: dict) -> BatchArrays:
    return BatchArrays(res["status"], res["objective"], res["x"], res["it1"], res["it2"])


# ---------------------------------------------------------------------------
# reference-compatible object API

class OutcomeList(Sequence):
    """``BatchReport.outcomes``: the per-LP ``SolveOutcome``s in input order, built from
    the packed result arrays when first read (then cached), so a 1e5-LP batch does not
    pay for 1e5 Python objects it may never look at.  Behaves as the reference's list
    (batch.py:172): len, indexing, slicing (-> list), iteration, equality with a list."""

    def __init__(self, res: dict):
        self._res = res
        self._cache: list[SolveOutcome | None] = [None] * len(res["status"])

    def __len__(self) -> int:
        return len(self._cache)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        if not 0 <= k < len(self):
            raise IndexError("outcome index out of range")
        o = self._cache[k]
        if o is None:
            o = self._cache[k] = outcome_from_arrays(self._res, k)
        return o

    def __iter__(self):
        step = 4096
        for s0 in range(0, len(self), step):
            s1 = min(len(self), s0 + step)
            if any(o is None for o in self._cache[s0:s1]):
                fresh = outcomes_from_arrays(self._res, s0, s1)
                for i, o in enumerate(fresh):
                    if self._cache[s0 + i] is None:
                        self._cache[s0 + i] = o
            yield from self._cache[s0:s1]

    def __eq__(self, other):
        if isinstance(other, (OutcomeList, list, tuple)):
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __repr__(self) -> str:
        return f"OutcomeList({len(self)} outcomes)"

    def status_counts(self) -> dict[str, int]:
        """Status.value -> count, keys in first-occurrence order (as the reference's loop)."""
        codes, first, counts = np.unique(self._res["status"], return_index=True, return_counts=True)
        order = np.argsort(first, kind="stable")
        return {STATUS_BY_CODE[int(codes[i])].value: int(counts[i]) for i in order}


def _solve_gather_sharded(ptrs: bytes, start: int, end: int, m: int, n: int, limits: SolverLimits,
                          devices: Sequence[int], out: dict) -> dict:
    """LPs [start, end) of a pointer table (blp_solve_batch_gather) into out[start:end],
    contiguous shards over `devices`, one host thread per device."""
    lim = limits.to_native()
    count = end - start
    sub = {k: v[start:end] for k, v in out.items()}
    devices = list(devices)[:max(1, count)]
    if len(devices) == 1 or count == 0:
        if count:
            _native.solve_gather(ptrs, count, m, n, lim, device=devices[0], out=sub, first=start)
        return sub
    errors: list[BaseException] = []

    def work(dev: int, s: int, e: int) -> None:
        try:
            _native.solve_gather(ptrs, e - s, m, n, lim, device=dev, out={k: v[s:e] for k, v in sub.items()},
                                 first=start + s)
        except BaseException as err:  # re-raised on the caller's thread
            errors.append(err)

    threads = [threading.Thread(target=work, args=(d, s, e))
               for d, (s, e) in zip(devices, shard_bounds(count, len(devices)))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return sub


def batch_solve(lps: Sequence[StandardFormLP], config: BatchConfig = BatchConfig()) -> BatchReport:
    """Solve every LP of a same-shaped batch on the GPU; outcomes land at their input index.

    Marshalling (SURVEY.md §7 hard part iv): one pass in C over the list (_pyobj.collect)
    takes each LP's A/b/c data pointers and the batch-worst artificial count; the library
    gathers the arrays with host threads into its pinned staging ring
    (blp_solve_batch_gather), pipelined with the copies and kernels; outcomes are built
    lazily (OutcomeList).  LPs whose arrays are not C-contiguous float64 numpy arrays are
    coerced here first.
    """
    from . import _pyobj
    lps = lps if isinstance(lps, list) else list(lps)
    if not lps:
        return BatchReport(outcomes=[], plan=plan_chunks(0, 1, config), chunk_seconds=[], total_seconds=0.0)
    m, n = lps[0].m, lps[0].n
    ptrs, slow, worst_artificial, first_hetero = _pyobj.collect(lps, m, n)
    if first_hetero >= 0:
        shapes = {(lp.m, lp.n) for lp in lps}
        raise HeterogeneousBatch(f"batch mixes LP shapes {sorted(shapes)}")
    count = len(lps)
    keep = []             # coerced copies of the slow LPs' arrays, alive until the solve returns
    bad_shape = -1        # the reference raises at the first invalid LP in index order
    if slow:
        table = np.frombuffer(ptrs, dtype=np.int64).reshape(3, count).copy()
        for k in slow:
            lp = lps[k]
            worst_artificial = max(worst_artificial, int(np.sum(np.asarray(lp.b, dtype=float) < 0)))
            if bad_shape >= 0:
                continue
            try:
                ok = np.shape(lp.A) == (m, n)
            except ValueError:  # ragged rows
                ok = False
            if not ok:
                bad_shape = k
                continue
            try:
                arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.float64)) for v in (lp.A, lp.b, lp.c)]
            except (TypeError, ValueError):   # non-numeric entries: validate() names them
                bad_shape = k
                continue
            keep.append(arrs)
            table[:, k] = [a.ctypes.data for a in arrs]
        ptrs = table.tobytes()
    lp_bytes = lp_memory_bytes(m, n, num_slack=m, num_artificial=worst_artificial,
                               data_size_bytes=config.data_size_bytes)
    plan = plan_chunks(count, lp_bytes, config)
    started = time.perf_counter()        # like batch.py:157, the timer covers everything after planning
    out = _native.alloc_outputs(count, n)
    if bad_shape >= 0:
        if bad_shape:
            res = _solve_gather_sharded(ptrs, 0, bad_shape, m, n, config.limits, config.devices, out)
            _raise_for_errors(res, lambda k: lps[k])
        raise ValueError(invalid_message(validate(lps[bad_shape])))
    # The plan's chunks (the reference's host-memory budget, batch.py:109-127) are solved in
    # one pipelined library call: the GPU path budgets device memory itself, and one call lets
    # the gather of later LPs overlap the kernels of earlier ones across chunk boundaries
    # (C3 through this API: 16 calls -> 1).  Each chunk's seconds are the batch's wall time
    # apportioned by chunk size; plan, chunk count and outcomes are the reference's.
    res = _solve_gather_sharded(ptrs, 0, count, m, n, config.limits, config.devices, out)
    _raise_for_errors(res, lambda k: lps[k])
    total = time.perf_counter() - started
    chunk_seconds = [total * (end - start) / count for start, end in plan.bounds]
    del keep
    return BatchReport(outcomes=OutcomeList(out), plan=plan, chunk_seconds=chunk_seconds, total_seconds=total)
