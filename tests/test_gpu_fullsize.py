"""Parity at BASELINE.json's full sizes: the exact inputs bench.py times (bench.workload),
solved through the public API, against the CPU oracle on every LP.

Bar (north star): status, x and per-phase iteration counts identical; objective within
1e-9 true relative error (golden_io.compare).  C3 is checked on its first 20,000 LPs by
default (the oracle needs ~1 ms per 100x100 two-phase LP and core); BLP_FULL_C3=1 checks
all 1e5.
"""
import os

import numpy as np
import pytest

from golden_io import compare

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _d(res):
    return dict(status=res.status, objective=res.objective, x=res.x, it1=res.iterations_phase1,
                it2=res.iterations_phase2)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_bench_workload_matches_oracle(cfg):
    import bench
    from oracle import oracle
    from paper_1802_08557_b200 import batch_solve_arrays, support_batch
    count = None
    if cfg == "c3" and os.environ.get("BLP_FULL_C3") != "1":
        count = 20_000
    A, b, c, shared, spec = bench.workload(cfg, count, 0)
    assert len(c) == (count or spec["count"])
    got = _d(support_batch(A, b, c) if shared else batch_solve_arrays(A, b, c))
    want = oracle.solve_batch(A, b, c, shared_Ab=shared, threads=oracle.host_cores())
    compare(got, want, f"{cfg} full size ({len(c)} LPs)")
    # the recipe's outcome mix is present at this size (not a degenerate all-one-status batch)
    kinds = set(np.unique(got["status"]).tolist())
    assert {"c1": {0}, "c2": {0, 2}, "c3": {0, 1, 2}, "c4": {0}, "c5": {0}}[cfg] <= kinds
