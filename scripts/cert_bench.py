"""Time batched certificates of GPU answers (host API: H2D + kernel + D2H).

    python scripts/cert_bench.py --config c2 --count 100000
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_1802_08557_b200 import batch_solve_arrays, support_batch  # noqa: E402
from paper_1802_08557_b200.certify import certify_batch  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2")
p.add_argument("--count", type=int, default=None)
a = p.parse_args()
A, b, c, shared, _ = bench.workload(a.config, a.count, 0)
res = support_batch(A, b, c) if shared else batch_solve_arrays(A, b, c)
certify_batch(A, b, c, res.x, res.status, shared_Ab=shared)      # warm-up
t = time.perf_counter()
cert = certify_batch(A, b, c, res.x, res.status, shared_Ab=shared)
dt = time.perf_counter() - t
opt = res.status == 0
print(json.dumps(dict(config=a.config, count=len(c), optimal=int(opt.sum()), certified=int(cert.certified[opt].sum()),
                      repriced=int(cert.repriced.sum()), seconds=dt, lps_per_s=len(c) / dt)))
