"""Device-resident timing of the reference's own random workload (gen_random_lps, feasible
start: single phase, few pivots) at the paper's sweep dims, dense family vs the lazy tableau.

    python scripts/lazy_vs_dense.py --dims 28 50 100 --count 20000
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08557_b200 import SolverLimits, _native, workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--dims", type=int, nargs="+", default=[28, 50, 100])
p.add_argument("--count", type=int, default=20000)
a = p.parse_args()
dev = torch.device("cuda:0")
for dim in a.dims:
    A, b, c = workloads.random_arrays(dim, a.count, seed=dim)
    tA, tb, tc = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (A, b, c))
    res = {}
    for mode in ("dense", "lazy"):
        os.environ["BLP_LAZY_SMALL"] = "0" if mode == "dense" else "1"   # dense family alone vs lazy-first
        out = dict(status=torch.empty(a.count, dtype=torch.int8, device=dev),
                   objective=torch.empty(a.count, dtype=torch.float64, device=dev),
                   x=torch.empty(a.count, dim, dtype=torch.float64, device=dev),
                   it1=torch.empty(a.count, dtype=torch.int32, device=dev),
                   it2=torch.empty(a.count, dtype=torch.int32, device=dev))
        lim = SolverLimits().to_native()
        _native.solve_device(tA, tb, tc, lim, out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _native.solve_device(tA, tb, tc, lim, out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[mode] = ({k: v.cpu().numpy() for k, v in out.items()}, statistics.median(ts), _native.kernel_variant(dim, dim))
    same = all(np.array_equal(res["dense"][0][k], res["lazy"][0][k]) for k in ("status", "it2", "x"))
    piv = res["dense"][0]["it2"].mean()
    print(json.dumps(dict(dim=dim, count=a.count, pivots=float(piv), dense=res["dense"][2], dense_ms=res["dense"][1],
                          lazy=res["lazy"][2], lazy_ms=res["lazy"][1], identical=bool(same))), flush=True)
