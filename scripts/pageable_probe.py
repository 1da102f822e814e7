"""e2e of batch_solve_arrays with ordinary (pageable) numpy inputs: the pinned staging ring.

    BLP_COPY_THREADS=8 BLP_STAGE_MB=64 python scripts/pageable_probe.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import time, os, numpy as np
from paper_1802_08557_b200 import batch_solve_arrays, workloads
A,b,c = workloads.afiro_arrays(100000)
batch_solve_arrays(A,b,c)
ts=[]
for _ in range(5):
    t=time.perf_counter(); batch_solve_arrays(A,b,c); ts.append(time.perf_counter()-t)
print(os.environ.get("BLP_COPY_THREADS"), os.environ.get("BLP_STAGE_MB"), "pageable C2 1e5 ms:", round(1e3*min(ts),1), os.cpu_count())
