"""e2e of one bench config through batch_solve_arrays / support_batch from pinned host buffers
(the bench.py e2e arm alone), median of K calls: A/B of library builds and knobs.

    BLP_LIBRARY=... python scripts/e2e_config.py --config c3 --count 50000 --steps 3
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_1802_08557_b200 import _native, batch_solve_arrays, support_batch  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c3")
p.add_argument("--count", type=int, default=None)
p.add_argument("--steps", type=int, default=3)
a = p.parse_args()
A, b, c, shared, spec = bench.workload(a.config, a.count, 0)
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
hA, hb, hc = pin(A), pin(b), pin(c)
call = (lambda: support_batch(hA, hb, hc)) if shared else (lambda: batch_solve_arrays(hA, hb, hc))
call()
ts = []
for _ in range(a.steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    call()
    ts.append(time.perf_counter() - t0)
ms = 1e3 * statistics.median(ts)
print(json.dumps({"config": a.config, "lib": str(_native.LIB_PATH.name), "e2e_ms": ms, "lps_per_s": len(hc) / ms * 1e3,
                  "all_ms": [round(1e3 * t, 2) for t in ts]}), flush=True)
