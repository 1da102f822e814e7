"""Time kernel variants on one config (device-resident, CUDA events, median of K launches).

    python scripts/sweep.py --config c2 --count 100000 --env BLP_RT_CPW=16 BLP_RT_CPW=32 BLP_KERNEL=smem
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
import bench  # noqa: E402
from paper_1802_08557_b200 import SolverLimits, _native  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2")
p.add_argument("--count", type=int, default=None)
p.add_argument("--steps", type=int, default=5)
p.add_argument("--env", nargs="*", default=[""])
p.add_argument("--max-iter", type=int, default=None, help="SolverLimits.max_iterations (per phase): isolates build cost")
p.add_argument("--shape", default=None, help="recipe:m:n instead of a config (afiro | degenerate | random)")
p.add_argument("--pipelined", action="store_true",
               help="time the steps back to back in one event region (host work overlaps, as in bench.py)")
a = p.parse_args()
if a.shape:
    from paper_1802_08557_b200 import workloads
    kind, sm, sn = a.shape.split(":")
    sm, sn, cnt0 = int(sm), int(sn), a.count or 100_000
    if kind == "afiro":
        A, b, c = workloads.afiro_arrays(cnt0, seed=9, m=sm, n=sn)
    elif kind == "degenerate":
        A, b, c = workloads.degenerate_arrays(cnt0, seed=9, m=sm, n=sn)
    else:
        A, b, c = workloads.random_arrays(max(sm, sn), cnt0, 9)
        A, b, c = A[:, :sm, :sn].copy(), b[:, :sm].copy(), c[:, :sn].copy()
    shared = False
    a.config = a.shape
else:
    A, b, c, shared, spec = bench.workload(a.config, a.count, 0)
dev = torch.device("cuda:0")
tA, tb, tc = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (A, b, c))
cnt, n = c.shape
m = b.shape[-1]
ref = None
for setting in a.env:
    saved = dict(os.environ)
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    out = dict(status=torch.empty(cnt, dtype=torch.int8, device=dev),
               objective=torch.empty(cnt, dtype=torch.float64, device=dev),
               x=torch.empty(cnt, n, dtype=torch.float64, device=dev),
               it1=torch.empty(cnt, dtype=torch.int32, device=dev),
               it2=torch.empty(cnt, dtype=torch.int32, device=dev))
    lim = SolverLimits(max_iterations=a.max_iter).to_native()
    _native.solve_device(tA, tb, tc, lim, out, shared_Ab=shared)
    torch.cuda.synchronize()
    ts = []
    if a.pipelined:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            _native.solve_device(tA, tb, tc, lim, out, shared_Ab=shared)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / a.steps)
    for _ in range(0 if a.pipelined else a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.solve_device(tA, tb, tc, lim, out, shared_Ab=shared)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res = {k: v.cpu().numpy() for k, v in out.items()}
    same = None
    if ref is None:
        ref = res
    else:
        same = all(np.array_equal(ref[k], res[k]) for k in ("status", "it1", "it2", "x"))
    ms = statistics.median(ts)
    piv = int((res["it1"].astype(np.int64) + res["it2"]).sum())
    print(json.dumps({"config": a.config, "env": setting, "variant": _native.kernel_variant(m, n, shared), "ms": ms,
                      "lps_per_s": cnt / ms * 1e3, "pivots_per_s": piv / ms * 1e3,
                      "gbs_alg": piv * bench.bytes_per_pivot(m, n) / ms / 1e6, "same_as_first": same}), flush=True)
    os.environ.clear()
    os.environ.update(saved)
