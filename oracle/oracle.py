"""ctypes front end of the C oracle (blp_oracle.c) -- TEST INFRASTRUCTURE ONLY.

The oracle is a plain-C restatement of the reference two-phase tableau
simplex (/root/reference/pkg/src/batchlp/tableau.py, simplex.py) with the
reference's full tableau layout, including artificial columns.  It is the
parity checker for the CUDA product path and the CPU baseline bench.py
reports; nothing in paper_1802_08557_b200/ may import it.

Pinned against the reference: tests/golden/ holds outcomes produced by the
imported reference (tests/golden/make_golden.py) and tests/test_oracle.py
checks this oracle against every one of them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

STATUS_NAMES = ("optimal", "unbounded", "infeasible", "iteration_limit",
                "error_phase1_unbounded", "error_nomem")


class _Limits(ctypes.Structure):
    _fields_ = [("max_iterations", ctypes.c_int32),
                ("anti_cycling", ctypes.c_int32),
                ("degenerate_limit", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_lib = None


def build() -> Path:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(LIB_PATH))
        f = lib.oracle_solve_batch
        P = ctypes.c_void_p
        f.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                      ctypes.POINTER(_Limits), P, P, P, P, P, ctypes.c_int32]
        f.restype = ctypes.c_int
        _lib = lib
    return _lib


def limits_struct(max_iterations=None, anti_cycling=True, degenerate_pivot_limit=None) -> _Limits:
    return _Limits(0 if max_iterations is None else int(max_iterations),
                   1 if anti_cycling else 0,
                   -1 if degenerate_pivot_limit is None else int(degenerate_pivot_limit), 0)


def solve_batch(A, b, c, *, shared_Ab: bool = False, max_iterations=None, anti_cycling=True,
                degenerate_pivot_limit=None, threads: int = 0) -> dict:
    """Solve a packed batch on the CPU.  A [B,m,n] (or [m,n] if shared_Ab), b [B,m] (or [m]), c [B,n].

    Returns dict(status int8 [B], objective f64 [B], x f64 [B,n], it1/it2 int32 [B], threads int).
    """
    lib = _load()
    c = np.ascontiguousarray(c, dtype=np.float64)
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    count, n = c.shape
    m = b.shape[-1]
    status = np.zeros(count, np.int8)
    objective = np.zeros(count, np.float64)
    x = np.zeros((count, n), np.float64)
    it1 = np.zeros(count, np.int32)
    it2 = np.zeros(count, np.int32)
    lim = limits_struct(max_iterations, anti_cycling, degenerate_pivot_limit)
    used = lib.oracle_solve_batch(A.ctypes.data, b.ctypes.data, c.ctypes.data, count, m, n,
                                  1 if shared_Ab else 0, ctypes.byref(lim), status.ctypes.data,
                                  objective.ctypes.data, x.ctypes.data, it1.ctypes.data,
                                  it2.ctypes.data, int(threads))
    return dict(status=status, objective=objective, x=x, it1=it1, it2=it2, threads=used)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def box_solve(lower, upper, direction) -> dict:
    """Hyper-rectangle LPs, restating boxlp.py:44-61 row by row (numpy, CPU): value (left-to-right
    sum; NaN if invalid), point (zeros if invalid), status (0 ok, -1 non-finite bound, k+1 first
    lower > upper, 1 when the only fault is lower+upper overflowing)."""
    lower = np.asarray(lower, np.float64)
    upper = np.asarray(upper, np.float64)
    direction = np.asarray(direction, np.float64)
    count, n = direction.shape
    value = np.full(count, np.nan)
    point = np.zeros((count, n))
    status = np.zeros(count, np.int32)
    for k in range(count):
        lo, hi, d = lower[k], upper[k], direction[k]
        with np.errstate(over="ignore", invalid="ignore"):
            ok = bool(((lo <= hi) & np.isfinite(lo + hi)).all())       # boxlp.py:51
        if not ok:
            if not (np.isfinite(lo).all() and np.isfinite(hi).all()):   # boxlp.py:58-59
                status[k] = -1
            else:
                status[k] = 1 + int(np.argmax(lo > hi))                  # boxlp.py:60
            continue
        p = np.where(d < 0, lo, hi)                                      # boxlp.py:53
        s = 0.0
        for j in range(n):
            s = s + d[j] * p[j]
        point[k] = p
        value[k] = s
    return dict(value=value, point=point, status=status)
