"""e2e (host buffers through batch_solve_arrays) vs sub-batch count: H2D/kernel/D2H overlap check."""
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08557_b200 import batch_solve_arrays, workloads  # noqa: E402

A, b, c = workloads.afiro_arrays(100_000)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
hA, hb, hc = pin(A), pin(b), pin(c)
for chunks in sys.argv[1:] or ["8", "16", "32"]:
    os.environ["BLP_HOST_CHUNKS"] = chunks
    batch_solve_arrays(hA, hb, hc)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch_solve_arrays(hA, hb, hc)
        ts.append(time.perf_counter() - t0)
    print(f"chunks={chunks} e2e_ms={1e3 * statistics.median(ts):.2f} min={1e3 * min(ts):.2f}", flush=True)
# pageable inputs for comparison
os.environ["BLP_HOST_CHUNKS"] = "16"
t0 = time.perf_counter(); batch_solve_arrays(A, b, c); print(f"pageable inputs: {1e3 * (time.perf_counter() - t0):.2f} ms")
