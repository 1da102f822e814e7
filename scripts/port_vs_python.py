"""The port-vs-Python factor: the reference package itself (pure Python,
imported read-only from /root/reference, batch_solve with W workers) against the C oracle
port (oracle/blp_oracle.c, the reference arm of bench.py) on the same LPs and host.
Run in the build container (the reference tree does not travel to the GPU box).

    python scripts/port_vs_python.py --config c2 --count 2000 --workers 1 8
"""
import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2")
p.add_argument("--count", type=int, default=2000)
p.add_argument("--workers", type=int, nargs="*", default=[1])
a = p.parse_args()

import batchlp  # noqa: E402  (the unmodified reference)
import bench  # noqa: E402
from oracle import oracle  # noqa: E402

A, b, c, shared, spec = bench.workload(a.config, a.count, 0)
lps = [batchlp.StandardFormLP(c=c[k], A=A if shared else A[k], b=b if shared else b[k]) for k in range(len(c))]
for w in a.workers:
    t0 = time.perf_counter()
    rep = batchlp.batch_solve(lps, batchlp.BatchConfig(worker_count=w))
    dt = time.perf_counter() - t0
    print(f"reference python batch_solve W={w}: {len(lps) / dt:.1f} LPs/s ({dt:.2f} s)")
    ref_status = [o.status.value for o in rep.outcomes]
for t in sorted({1, *a.workers}):
    t0 = time.perf_counter()
    res = oracle.solve_batch(A, b, c, shared_Ab=shared, threads=t)
    dt = time.perf_counter() - t0
    print(f"C port (oracle) threads={t}: {len(lps) / dt:.1f} LPs/s ({dt:.3f} s)")
names = {0: "optimal", 1: "unbounded", 2: "infeasible", 3: "iteration_limit"}
assert [names[int(s)] for s in res["status"]] == ref_status, "port and reference disagree"
print(f"cores here: {len(os.sched_getaffinity(0))}")
