"""Synthetic LP workloads: the reference generator and the SURVEY.md §8(d) recipes.

``gen_random_lps`` reproduces /root/reference/pkg/src/batchlp/generate.py:15-35
draw-for-draw (per LP: A, then b, then c from one ``default_rng(seed)``), so a
seed gives the same LPs as the reference.  ``random_arrays`` is the same
stream written straight into packed arrays.

The other generators are vectorised recipes for the benchmark configurations
(BASELINE.json "configs"); each returns packed fp64 arrays (A [B,m,n],
b [B,m], c [B,n]) and documents its draw order, which is part of the recipe.
All coefficients are small integers or fixed-precision draws stored as fp64,
and b = A.x0 + s is exact in fp64 for the integer recipes.
"""
from __future__ import annotations

import numpy as np

from .model import StandardFormLP

# Beale's cycling instance (the reference's anti-cycling test LP).
BEALE_A = np.array([[0.25, -60.0, -0.04, 9.0],
                    [0.5, -90.0, -0.02, 3.0],
                    [0.0, 0.0, 1.0, 0.0]])
BEALE_B = np.array([0.0, 0.0, 1.0])
BEALE_C = np.array([0.75, -150.0, 0.02, -6.0])


def gen_random_lps(dim: int, count: int, seed: int, feasible_start: bool = True) -> list[StandardFormLP]:
    """``count`` square LPs of size ``dim`` (generate.py:15-35): A,b in [1,1000], c in [1,500]."""
    A, b, c = random_arrays(dim, count, seed, feasible_start)
    return [StandardFormLP(c=c[k], A=A[k], b=b[k]) for k in range(count)]


def random_arrays(dim: int, count: int, seed: int, feasible_start: bool = True):
    """Packed form of gen_random_lps (same RNG stream, same values)."""
    if dim < 1:
        raise ValueError("dim must be >= 1")
    if count < 0:
        raise ValueError("count must be >= 0")
    rng = np.random.default_rng(seed)
    A = np.empty((count, dim, dim))
    b = np.empty((count, dim))
    c = np.empty((count, dim))
    for k in range(count):
        A[k] = rng.integers(1, 1001, size=(dim, dim))
        b[k] = rng.integers(1, 1001, size=dim)
        c[k] = rng.integers(1, 501, size=dim)
    if not feasible_start:
        b = -b
    return A, b, c


def _infeasible_rows(rng, A, b, mask):
    """Row k := -row 0 with b_k = -b_0 - 1 on the masked LPs: A0.x <= b0 and A0.x >= b0+1."""
    count, m, _ = A.shape
    k = rng.integers(1, m, size=count)
    idx = np.flatnonzero(mask)
    A[idx, k[idx], :] = -A[idx, 0, :]
    b[idx, k[idx]] = -b[idx, 0] - 1.0


def afiro_arrays(count: int = 100_000, seed: int = 2, m: int = 28, n: int = 32, infeasible_frac: float = 0.10):
    """C2: afiro-shaped two-phase LPs with mixed-sign b.

    Draw order: A ~ U{-50..50} [B,m,n]; row 0 redrawn U{1..50} (bounds every
    variable); x0 ~ U{1..4} [B,n]; s ~ U{1..19} [B,m]; b = A.x0 + s; c ~
    U{-20..50} [B,n]; u ~ U[0,1) [B]; k ~ U{1..m-1} [B]; LPs with u <
    infeasible_frac get row k = -row 0, b_k = -b_0 - 1 (infeasible).
    """
    rng = np.random.default_rng(seed)
    A = rng.integers(-50, 51, size=(count, m, n)).astype(np.float64)
    A[:, 0, :] = rng.integers(1, 51, size=(count, n))
    x0 = rng.integers(1, 5, size=(count, n)).astype(np.float64)
    s = rng.integers(1, 20, size=(count, m)).astype(np.float64)
    b = np.einsum("kij,kj->ki", A, x0) + s
    c = rng.integers(-20, 51, size=(count, n)).astype(np.float64)
    u = rng.random(count)
    _infeasible_rows(rng, A, b, u < infeasible_frac)
    return A, b, c


def padded_beale(m: int, n: int):
    """Beale's 3x4 cycling block padded to (m, n): rows 3.. bound x_4.. by 1, c_pad = -1."""
    A = np.zeros((m, n))
    b = np.zeros(m)
    c = np.zeros(n)
    A[:3, :4] = BEALE_A
    b[:3] = BEALE_B
    c[:4] = BEALE_C
    pad = n - 4
    for k in range(3, m):
        A[k, 4 + (k - 3) % pad] = 1.0
        b[k] = 1.0
    c[4:] = -1.0
    return A, b, c


def degenerate_arrays(count: int = 100_000, seed: int = 3, m: int = 100, n: int = 100):
    """C3: 100x100 degenerate mix with unbounded, infeasible and padded-Beale LPs.

    Draw order: A ~ U{-3..3}; row 0 redrawn U{1..3}; c ~ U{-3..3}; u ~ U[0,1);
    LPs with u < 0.10 become unbounded (column 0 := -|column 0|, A[0,0] = -1,
    c_0 = 5, before b is formed); x0 ~ U{0,1} [B,n]; s ~ U{0,1} [B,m] (zero
    slacks make the start degenerate); b = A.x0 + s; k ~ U{1..m-1}: LPs with
    0.10 <= u < 0.20 get the infeasible row pair; LPs with 0.20 <= u < 0.21
    are replaced by the padded Beale instance (forces the Bland switch).
    """
    rng = np.random.default_rng(seed)
    A = rng.integers(-3, 4, size=(count, m, n)).astype(np.float64)
    A[:, 0, :] = rng.integers(1, 4, size=(count, n))
    c = rng.integers(-3, 4, size=(count, n)).astype(np.float64)
    u = rng.random(count)
    unb = u < 0.10
    A[unb, :, 0] = -np.abs(A[unb, :, 0])
    A[unb, 0, 0] = -1.0
    c[unb, 0] = 5.0
    x0 = rng.integers(0, 2, size=(count, n)).astype(np.float64)
    s = rng.integers(0, 2, size=(count, m)).astype(np.float64)
    b = np.einsum("kij,kj->ki", A, x0) + s
    _infeasible_rows(rng, A, b, (u >= 0.10) & (u < 0.20))
    beale = np.flatnonzero((u >= 0.20) & (u < 0.21))
    if beale.size:
        Ab, bb, cb = padded_beale(m, n)
        A[beale], b[beale], c[beale] = Ab, bb, cb
    return A, b, c


def support_polytope(seed: int = 4, m: int = 64, n: int = 32):
    """C4 polytope: A ~ U(-1,1) + 2I on the first n rows, last row all ones; b ~ U(1,2), b_last = 1e3."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, size=(m, n))
    A[:n] += 2.0 * np.eye(n)
    A[m - 1] = 1.0
    b = rng.uniform(1.0, 2.0, size=m)
    b[m - 1] = 1e3
    return A, b


def support_polytope_two_phase(seed: int = 44, m: int = 64, n: int = 32, lower: int = 16):
    """C4b: the C4 polytope with `lower` lower-bound rows, so b has negative entries and every
    direction needs phase 1 -- the same phase 1 for all of them.

    Draw order: A ~ U(-1,1) [m,n]; b ~ U(1,2) [m]; t ~ U(0.01,0.02) [lower].  Then A[:n] += 2I;
    rows n..n+lower-1 become -e_k (k < lower) with b = -t_k (x_k >= t_k); the last row is all
    ones with b = 1e3.  x = 0.02 on the first `lower` coordinates (0 elsewhere) is feasible.
    """
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, size=(m, n))
    b = rng.uniform(1.0, 2.0, size=m)
    t = rng.uniform(0.01, 0.02, size=lower)
    A[:n] += 2.0 * np.eye(n)
    for k in range(lower):
        A[n + k] = 0.0
        A[n + k, k] = -1.0
        b[n + k] = -t[k]
    A[m - 1] = 1.0
    b[m - 1] = 1e3
    return A, b


def support_directions(count: int = 1_000_000, seed: int = 4, n: int = 32, offset: int = 0):
    """C4 directions: C ~ N(0,1) [count, n], drawn after the polytope from the same seed."""
    rng = np.random.default_rng(seed)
    rng.uniform(-1.0, 1.0, size=(64, n))   # polytope draws come first
    rng.uniform(1.0, 2.0, size=64)
    if offset:
        rng.standard_normal((offset, n))
    return rng.standard_normal((count, n))


def big_arrays(count: int = 10_000, seed: int = 5, dim: int = 500):
    """C5: gen_random_lps(500, count, seed=5) packed (feasible start; 4 MB tableaux, beyond one SM)."""
    return random_arrays(dim, count, seed, True)


def big_two_phase_arrays(count: int = 4, seed: int = 55, dim: int = 500):
    """C5b: the C2 recipe at dim x dim (two-phase, ~12k pivots per LP)."""
    return afiro_arrays(count, seed, dim, dim)


CONFIGS = {
    "c1": dict(m=5, n=5, count=1_000, doc="gen_random_lps(5, 1000, seed=0), single phase"),
    "c2": dict(m=28, n=32, count=100_000, doc="afiro-shaped 28x32 two-phase, mixed-sign b, seed 2"),
    "c3": dict(m=100, n=100, count=100_000, doc="100x100 degenerate mix + Bland, seed 3"),
    "c4": dict(m=64, n=32, count=1_000_000, doc="support function: one 64x32 polytope, 1e6 directions, seed 4"),
    "c5": dict(m=500, n=500, count=10_000, doc="gen_random_lps(500, 1e4, seed=5), 4 MB tableaux (cluster-resident)"),
    # stress variants (not BASELINE.json configs): C4 with a shared phase 1, C5 two-phase
    "c4b": dict(m=64, n=32, count=1_000_000,
                doc="support function, two-phase: 64x32 polytope with 16 b < 0 rows (seed 44), 1e6 directions"),
    "c5b": dict(m=500, n=500, count=8, doc="C2 recipe at 500x500, seed 55 (two-phase, ~12k pivots per LP)"),
}


def make_config(name: str, count: int | None = None, offset: int = 0):
    """Packed (A, b, c, shared_Ab) for a named config; count overrides the default size."""
    spec = CONFIGS[name]
    cnt = spec["count"] if count is None else count
    if name == "c1":
        A, b, c = random_arrays(5, cnt, 0)
        return A, b, c, False
    if name == "c2":
        A, b, c = afiro_arrays(cnt)
        return A, b, c, False
    if name == "c3":
        A, b, c = degenerate_arrays(cnt)
        return A, b, c, False
    if name == "c4":
        A, b = support_polytope()
        return A, b, support_directions(cnt, offset=offset), True
    if name == "c5":
        A, b, c = big_arrays(cnt)
        return A, b, c, False
    if name == "c4b":
        A, b = support_polytope_two_phase()
        return A, b, support_directions(cnt, offset=offset), True
    if name == "c5b":
        A, b, c = big_two_phase_arrays(cnt)
        return A, b, c, False
    raise KeyError(name)
