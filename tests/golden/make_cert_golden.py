"""Golden certificates from the REFERENCE's check_certificate.

Run in the build container (where /root/reference exists), after make_golden.py:

    python tests/golden/make_cert_golden.py

For the packed golden families (inputs regenerated from their recipes, points =
the reference's own optimal outcomes stored in tests/golden/<stem>.npz), and
for perturbed / fake points of the C2 family, it records the reference's
Certificate fields and whether its complementary-prices search
(oracle.py:226-242) ran.  A seeded search over small degenerate LPs collects
instances whose basis route fails, so the prices path is pinned too.
Output: tests/golden/cert/<name>.npz.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

from batchlp import SolveOutcome, Status, solve, standard_form  # noqa: E402  (the reference)
from batchlp import oracle as ref_oracle  # noqa: E402

from golden_io import packed_fixture  # noqa: E402

OUT = HERE / "cert"
_calls = []
_orig = ref_oracle._complementary_prices


def _traced(*a, **k):
    _calls.append(1)
    return _orig(*a, **k)


ref_oracle._complementary_prices = _traced


def certify(A, b, c, x):
    _calls.clear()
    cert = ref_oracle.check_certificate(standard_form(c, A, b), SolveOutcome(Status.OPTIMAL, 0.0, x))
    return cert.max_reduced_cost, cert.max_violation, cert.max_negativity, cert.certified, bool(_calls)


def table(rows):
    rc, viol, neg, ok, pr = (np.array(v) for v in zip(*rows))
    return dict(max_reduced_cost=rc.astype(float), max_violation=viol.astype(float),
                max_negativity=neg.astype(float), certified=ok.astype(bool), prices=pr.astype(bool))


def family(stem: str, limit: int):
    fx = packed_fixture(stem)
    opt = np.flatnonzero(fx["status"] == 0)[:limit]
    A, b = fx["A"], fx["b"]
    rows = [certify(A if fx["shared"] else A[k], b if fx["shared"] else b[k], fx["c"][k], fx["x"][k])
            for k in opt]
    np.savez_compressed(OUT / f"{stem}.npz", source=stem, idx=opt, **table(rows))
    t = table(rows)
    print(stem, len(opt), "certified", int(t["certified"].sum()), "prices", int(t["prices"].sum()), flush=True)


def fakes():
    """Perturbed points of C2 LPs: violations, negativity, sub-optimality."""
    fx = packed_fixture("c2_afiro")
    rng = np.random.default_rng(4242)
    opt = np.flatnonzero(fx["status"] == 0)[:300]
    xs, rows = [], []
    for j, k in enumerate(opt):
        x = fx["x"][k].copy()
        kind = j % 5
        if kind == 0:
            x = x + rng.uniform(-1e-3, 1e-3, x.shape)
        elif kind == 1:
            x = x * 0.9
        elif kind == 2:
            x = np.zeros_like(x)
        elif kind == 3:
            x[int(rng.integers(0, len(x)))] = -0.25
        else:
            x = x + 1e-9 * rng.standard_normal(x.shape)
        xs.append(x)
        rows.append(certify(fx["A"][k], fx["b"][k], fx["c"][k], x))
    np.savez_compressed(OUT / "c2_fakes.npz", source="c2_afiro", idx=opt, x=np.array(xs), **table(rows))
    t = table(rows)
    print("c2_fakes", len(opt), "certified", int(t["certified"].sum()), "prices", int(t["prices"].sum()))


def price_cases(want: int = 40, seed: int = 777):
    """Small degenerate LPs whose greedy basis is dual-infeasible (the prices path)."""
    rng = np.random.default_rng(seed)
    As, bs, cs, xs, rows = [], [], [], [], []
    m, n = 6, 5
    tries = 0
    while len(rows) < want and tries < 200000:
        tries += 1
        A = rng.integers(-2, 3, size=(m, n)).astype(float)
        A[0] = rng.integers(1, 3, size=n)
        b = rng.integers(0, 2, size=m).astype(float) * rng.integers(0, 3, size=m)
        c = rng.integers(-2, 4, size=n).astype(float)
        out = solve(standard_form(c, A, b))
        if not out.is_optimal():
            continue
        r = certify(A, b, c, out.primal_point)
        if r[4]:
            As.append(A), bs.append(b), cs.append(c), xs.append(out.primal_point), rows.append(r)
    np.savez_compressed(OUT / "prices_small.npz", source="explicit", A=np.array(As), b=np.array(bs),
                        c=np.array(cs), x=np.array(xs), **table(rows))
    t = table(rows)
    print("prices_small", len(rows), "of", tries, "tries; certified", int(t["certified"].sum()))


def main():
    OUT.mkdir(exist_ok=True)
    price_cases()
    fakes()
    for stem, limit in (("c1_rand5", 1000), ("c2_afiro", 2000), ("afiro_m12_n8", 1500), ("afiro_m45_n30", 400),
                        ("c4_support", 2000), ("c3_degenerate", 150), ("afiro_m20_n400", 60)):
        family(stem, limit)


if __name__ == "__main__":
    main()
