"""Small batch of one kernel family for compute-sanitizer (racecheck / synccheck /
memcheck on the shared-memory kernels).  Host buffers (no torch), checked against the oracle.

    compute-sanitizer --tool racecheck python scripts/san_run.py condensed_c2
    BLP_LAZY_WS=1 compute-sanitizer --tool synccheck python scripts/san_run.py lazy_150

The family is picked by shape and the BLP_* environment knobs the case sets (blp_capi.cu
plan_launch), so every kernel of the default plan and the opt-in forms is reachable.
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

# name: (generator, env knobs); generators are the workloads recipes at small counts
CASES = {
    "condensed_c2": ("afiro:28:32:64", {}),
    "condensed_c2_direct": ("afiro:28:32:64", {"BLP_CT_STAGE": "0"}),
    "condensed_stage_short": ("afiro:20:10:64", {"BLP_CT_STAGE": "2"}),
    "condensed_narrow": ("afiro:64:8:64", {}),
    "condensed_c4": ("support:64", {}),
    "warplp2_c2": ("afiro:28:32:64", {"BLP_CONDENSED": "0"}),
    "warplp_c1": ("random:5:64", {"BLP_CONDENSED": "0"}),
    "pairlp_c4": ("afiro:64:32:24", {"BLP_CONDENSED": "0", "BLP_LAZY_SMALL": "0"}),
    "quadlp_c3": ("c3:8", {"BLP_LAZY_SMALL": "0", "BLP_CMULTI": "0"}),
    "cmulti_c3": ("c3:8", {"BLP_LAZY_SMALL": "0"}),
    "cmulti_lazy_c3": ("c3:8", {}),
    "cmulti_c4": ("afiro:64:32:24", {"BLP_CMULTI": "3", "BLP_LAZY_SMALL": "0"}),
    "condensed_p1": ("support2:64", {}),
    "lazy_c3": ("random:100:12", {}),
    "lazy_support": ("support:64", {"BLP_CONDENSED": "0"}),
    "lazy_150": ("random:150:6", {}),
    "lazy_150_ws": ("random:150:6", {"BLP_LAZY_WS": "1"}),
    "cluster_150": ("afiro:150:150:3", {}),
    "hbm_150": ("afiro:150:150:2", {"BLP_FORCE_HBM": "1"}),
}


def make(spec: str):
    from paper_1802_08557_b200 import workloads
    kind, *a = spec.split(":")
    if kind == "afiro":
        m, n, cnt = map(int, a)
        return (*workloads.afiro_arrays(cnt, seed=11, m=m, n=n), False)
    if kind == "random":
        dim, cnt = map(int, a)
        return (*workloads.random_arrays(dim, cnt, seed=12), False)
    if kind == "c3":
        return (*workloads.degenerate_arrays(int(a[0]), seed=3), False)
    if kind == "support2":
        A, b = workloads.support_polytope_two_phase()
        return A, b, workloads.support_directions(int(a[0])), True
    if kind == "support":
        A, b = workloads.support_polytope()
        return A, b, workloads.support_directions(int(a[0])), True
    raise ValueError(spec)


def main():
    name = sys.argv[1]
    spec, env = CASES[name]
    os.environ.update(env)
    from oracle import oracle
    from paper_1802_08557_b200 import _native, batch_solve_arrays, support_batch
    A, b, c, shared = make(spec)
    got = support_batch(A, b, c) if shared else batch_solve_arrays(A, b, c)
    want = oracle.solve_batch(A, b, c, shared_Ab=shared)
    ok = (np.array_equal(got.status, want["status"]) and np.array_equal(got.x, want["x"])
          and np.array_equal(got.iterations_phase1, want["it1"]) and np.array_equal(got.iterations_phase2, want["it2"]))
    m, n = b.shape[-1], c.shape[1]
    print(f"{name}: {len(c)} LPs {m}x{n} via {_native.kernel_variant(m, n)} parity={'ok' if ok else 'MISMATCH'}")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
