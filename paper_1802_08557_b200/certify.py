"""Batched optimality certificates on the GPU.

Mirrors the reference's ``Certificate`` / ``check_certificate``
(/root/reference/pkg/src/batchlp/oracle.py:22-44,168-242) for whole batches:
``certify_batch`` checks every OPTIMAL outcome of a packed batch from A, b,
c and the point alone (libblp's ``blp_certify_batch_host``: primal residual,
negativity, a basis rebuilt from the point's support and its duals), so 1e5-1e6
GPU answers are verified at GPU speed instead of with the per-LP Python oracle.

Where the basis route leaves a positive reduced cost on a primal-feasible
point (degenerate optima), the reference searches for complementary-slackness
prices with HiGHS (oracle.py:226-242).  Here that auxiliary LP is formed for
the flagged LPs only and solved by the batched simplex itself; feasible
prices re-price the LP on the GPU (``blp_certify_reprice_host``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .model import SolveOutcome, StandardFormLP

ORACLE_TOL = 1e-7   # oracle.py:22, looser than the solver's 1e-9 to absorb elimination round-off


@dataclass(frozen=True)
class Certificate:
    """From-scratch optimality evidence for a claimed Optimal outcome (oracle.py:30-44)."""

    max_reduced_cost: float
    max_violation: float
    max_negativity: float
    tolerance: float = ORACLE_TOL

    @property
    def certified(self) -> bool:
        return (self.max_reduced_cost <= self.tolerance
                and self.max_violation <= self.tolerance
                and self.max_negativity <= self.tolerance)


@dataclass
class CertificateBatch:
    """Per-LP certificate fields (NaN where the outcome is not OPTIMAL)."""

    max_reduced_cost: np.ndarray
    max_violation: np.ndarray
    max_negativity: np.ndarray
    repriced: np.ndarray        # bool: complementary prices replaced the basis-route value
    tolerance: float = ORACLE_TOL

    @property
    def certified(self) -> np.ndarray:
        t = self.tolerance
        return (self.max_reduced_cost <= t) & (self.max_violation <= t) & (self.max_negativity <= t)

    def certificate(self, k: int) -> Certificate:
        return Certificate(float(self.max_reduced_cost[k]), float(self.max_violation[k]),
                           float(self.max_negativity[k]), self.tolerance)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def price_lps(A, b, c, x, tol: float, *, shared_Ab: bool = False):
    """The complementary-prices feasibility LPs (oracle.py:226-242) in the solver's standard form.

    Variables y (m), y >= 0.  Rows, 2n + m of them so every LP of the batch has
    one shape: for a support column j (x_j > tol) A_j.y <= c_j and
    -A_j.y <= -c_j; for a loose column -A_j.y <= -c_j and an empty row; for a
    slack row i with level b_i - A_i.x > tol the bound y_i <= 0 (y_i fixed at
    0), else an empty row.  Zero objective: OPTIMAL <=> such prices exist.
    """
    count, n = c.shape
    m = b.shape[-1]
    Ab = np.broadcast_to(A, (count, m, n)) if shared_Ab else A
    bb = np.broadcast_to(b, (count, m)) if shared_Ab else b
    level_slack = bb - np.einsum("kij,kj->ki", Ab, x)
    support = x > tol
    At = np.swapaxes(Ab, 1, 2)                                   # [count, n, m]
    P = np.zeros((count, 2 * n + m, m))
    h = np.zeros((count, 2 * n + m))
    P[:, 0:2 * n:2] = np.where(support[:, :, None], At, -At)
    h[:, 0:2 * n:2] = np.where(support, c, -c)
    P[:, 1:2 * n:2] = np.where(support[:, :, None], -At, 0.0)
    h[:, 1:2 * n:2] = np.where(support, -c, 0.0)
    slack_pos = level_slack > tol                                # basic slack -> price fixed at 0
    rows = 2 * n + np.arange(m)
    P[:, rows, np.arange(m)] = np.where(slack_pos, 1.0, 0.0)
    return P, h, np.zeros((count, m))


def certify_batch(A, b, c, x, status, tol: float = ORACLE_TOL, *, shared_Ab: bool = False,
                  device: int = 0) -> CertificateBatch:
    """Certificates for every OPTIMAL (status 0) LP of a packed batch.

    A [B,m,n] (or [m,n] with shared_Ab), b [B,m] (or [m]), c [B,n], x [B,n], status [B].
    """
    A, b, c, x = _f64(A), _f64(b), _f64(c), _f64(x)
    status = np.ascontiguousarray(status, dtype=np.int8)
    out = _native.certify_host(A, b, c, x, status, tol, shared_Ab=shared_Ab, device=device)
    need = out["needs_prices"].astype(bool)
    repriced = np.zeros(len(c), dtype=bool)
    if need.any():
        from .batch import batch_solve_arrays
        idx = np.flatnonzero(need)
        Asub = A if shared_Ab else A[idx]
        bsub = b if shared_Ab else b[idx]
        P, h, z = price_lps(Asub, bsub, c[idx], x[idx], tol, shared_Ab=shared_Ab)
        res = batch_solve_arrays(P, h, z, devices=(device,))
        found = res.status == 0
        if found.any():
            mask = np.zeros(len(c), np.int8)
            mask[idx[found]] = 1
            y = np.zeros((len(c), b.shape[-1]))
            y[idx[found]] = res.x[found]
            _native.certify_reprice_host(A, c, y, mask, out["max_reduced_cost"], shared_Ab=shared_Ab,
                                         device=device)
            repriced[idx[found]] = True
    return CertificateBatch(out["max_reduced_cost"], out["max_violation"], out["max_negativity"], repriced, tol)


def check_certificate(lp: StandardFormLP, outcome: SolveOutcome, tol: float = ORACLE_TOL) -> Certificate:
    """One LP through the batched path (same contract as oracle.py:168-223)."""
    if not outcome.is_optimal():
        raise ValueError("certificate checks apply to Optimal outcomes only")
    m, n = lp.m, lp.n
    A = _f64(lp.A).reshape(1, m, n)
    x = _f64(outcome.primal_point).reshape(1, n)
    res = certify_batch(A, _f64(lp.b).reshape(1, m), _f64(lp.c).reshape(1, n), x, np.zeros(1, np.int8), tol)
    return res.certificate(0)
