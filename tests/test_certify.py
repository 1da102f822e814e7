"""Batched GPU certificates vs the reference's check_certificate.

Golden values: tests/golden/make_cert_golden.py (the reference on its own optimal
points, perturbed points, and degenerate LPs that take its complementary-prices
route).  Bar: the certified verdict and the prices route identical; violation and
negativity to 1e-12 (same sums, different order); reduced cost to 1e-9 where both
take the basis route (QR duals vs LU duals of the same basis), <= tol after prices.
"""
from pathlib import Path

import numpy as np
import pytest

from golden_io import GOLDEN, packed_fixture

CERT = GOLDEN / "cert"
torch = pytest.importorskip("torch")


def _case(name):
    z = np.load(CERT / f"{name}.npz", allow_pickle=False)
    src = str(z["source"])
    if src == "explicit":
        A, b, c, x = z["A"], z["b"], z["c"], z["x"]
        shared = False
    else:
        fx = packed_fixture(src)
        idx = z["idx"]
        shared = fx["shared"]
        A = fx["A"] if shared else fx["A"][idx]
        b = fx["b"] if shared else fx["b"][idx]
        c = fx["c"][idx]
        x = z["x"] if "x" in z.files else fx["x"][idx]
    return dict(A=A, b=b, c=c, x=x, shared=shared, **{k: z[k] for k in
                ("max_reduced_cost", "max_violation", "max_negativity", "certified", "prices")})


def _names():
    return sorted(p.stem for p in CERT.glob("*.npz"))


# ---- CPU: the auxiliary prices LP is formed as the reference's linprog call states it

def test_price_lps_form_the_reference_feasibility_problem():
    from oracle import oracle
    from paper_1802_08557_b200.certify import ORACLE_TOL, price_lps
    cs = _case("prices_small")
    P, h, z = price_lps(cs["A"], cs["b"], cs["c"], cs["x"], ORACLE_TOL)
    m, n = cs["b"].shape[1], cs["c"].shape[1]
    assert P.shape == (len(cs["c"]), 2 * n + m, m) and h.shape == (len(cs["c"]), 2 * n + m)
    res = oracle.solve_batch(P, h, z)           # the CPU oracle solves the same LPs (test infra)
    assert (res["status"] == 0).all()           # the reference found prices for every case
    for k in range(len(cs["c"])):
        A, b, c, x, y = cs["A"][k], cs["b"][k], cs["c"][k], cs["x"][k], res["x"][k]
        support = x > ORACLE_TOL
        slack_pos = (b - A @ x) > ORACLE_TOL
        assert (y >= 0).all() and (y[slack_pos] == 0).all()
        assert np.allclose(A.T[support] @ y, c[support], atol=1e-9)
        assert (A.T[~support] @ y >= c[~support] - 1e-9).all()


def test_certificate_semantics():
    from paper_1802_08557_b200.certify import Certificate
    assert Certificate(1e-7, 0.0, 0.0).certified
    assert not Certificate(1.1e-7, 0.0, 0.0).certified
    assert not Certificate(0.0, 0.0, 2e-7, tolerance=1e-7).certified


# ---- GPU parity

@pytest.mark.gpu
@pytest.mark.parametrize("name", _names())
def test_certify_batch_matches_reference(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_08557_b200.certify import certify_batch
    cs = _case(name)
    got = certify_batch(cs["A"], cs["b"], cs["c"], cs["x"], np.zeros(len(cs["c"]), np.int8),
                        shared_Ab=cs["shared"])
    assert np.array_equal(got.certified, cs["certified"]), name
    assert np.array_equal(got.repriced, cs["prices"]), name
    scale = np.maximum(1.0, np.abs(cs["max_violation"]))
    assert (np.abs(got.max_violation - cs["max_violation"]) <= 1e-12 * scale * 1e3).all(), name
    assert np.array_equal(got.max_negativity, cs["max_negativity"]), name
    basis = ~cs["prices"]
    d = np.abs(got.max_reduced_cost - cs["max_reduced_cost"])[basis]
    assert (d <= 1e-9 * np.maximum(1.0, np.abs(cs["max_reduced_cost"][basis]))).all(), (name, d.max())
    assert (got.max_reduced_cost[cs["prices"]] <= got.tolerance).all() == bool(cs["certified"][cs["prices"]].all())


@pytest.mark.gpu
def test_check_certificate_known_answers():
    """oracle.py contract on the reference's WORKSHOP LP (test_oracle.py:72-105)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_08557_b200 import SolveOutcome, Status, solve, standard_form
    from paper_1802_08557_b200.certify import check_certificate
    lp = standard_form([3.0, 5.0], [[1, 0], [0, 2], [3, 2]], [4.0, 12.0, 18.0])
    cert = check_certificate(lp, solve(lp))
    assert cert.certified and cert.max_reduced_cost <= 1e-9
    assert cert.max_violation == 0.0 and cert.max_negativity == 0.0
    cert = check_certificate(lp, SolveOutcome(Status.OPTIMAL, 36.3, np.array([2.1, 6.0])))
    assert cert.max_violation == pytest.approx(0.3) and not cert.certified
    cert = check_certificate(lp, SolveOutcome(Status.OPTIMAL, 0.0, np.array([0.0, 0.0])))
    assert cert.max_violation == 0.0 and cert.max_negativity == 0.0
    assert cert.max_reduced_cost == pytest.approx(5.0) and not cert.certified
    cert = check_certificate(lp, SolveOutcome(Status.OPTIMAL, 0.0, np.array([-0.5, 0.0])))
    assert cert.max_negativity == pytest.approx(0.5)
    with pytest.raises(ValueError, match="Optimal outcomes only"):
        check_certificate(lp, SolveOutcome(Status.UNBOUNDED))


@pytest.mark.gpu
def test_certify_full_c2_batch_of_gpu_answers():
    """The §8(f) use: verify 1e5 GPU answers at GPU speed; every optimal C2 answer certifies."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_08557_b200 import batch_solve_arrays, workloads
    from paper_1802_08557_b200.certify import certify_batch
    A, b, c = workloads.afiro_arrays(100_000)
    res = batch_solve_arrays(A, b, c)
    cert = certify_batch(A, b, c, res.x, res.status)
    opt = res.status == 0
    assert cert.certified[opt].all()
    assert np.isnan(cert.max_reduced_cost[~opt]).all()
