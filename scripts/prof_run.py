"""Minimal driver for ncu captures: N launches of the solver on one config (device-resident inputs).

    ncu ... python scripts/prof_run.py --config c2 --count 20000 --launches 2
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_1802_08557_b200 import SolverLimits, _native  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2")
p.add_argument("--count", type=int, default=20000)
p.add_argument("--launches", type=int, default=2)
a = p.parse_args()
A, b, c, shared, _ = bench.workload(a.config, a.count, 0)
dev = torch.device("cuda:0")
tA, tb, tc = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (A, b, c))
cnt, n = c.shape
out = dict(status=torch.empty(cnt, dtype=torch.int8, device=dev),
           objective=torch.empty(cnt, dtype=torch.float64, device=dev),
           x=torch.empty(cnt, n, dtype=torch.float64, device=dev),
           it1=torch.empty(cnt, dtype=torch.int32, device=dev),
           it2=torch.empty(cnt, dtype=torch.int32, device=dev))
for _ in range(a.launches):
    _native.solve_device(tA, tb, tc, SolverLimits().to_native(), out, shared_Ab=shared)
torch.cuda.synchronize()
piv = (out["it1"].long() + out["it2"].long()).sum().item()
print(f"{a.config} count={cnt} kernel={_native.kernel_variant(b.shape[-1], n)} pivots/launch={piv}")
