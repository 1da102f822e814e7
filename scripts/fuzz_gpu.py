"""Randomised parity sweep (GPU vs the CPU oracle) for a fixed wall-clock budget: random
shapes, LP recipes, solver limits, kernel families and the support-function mode.  Prints
one line per case and a summary; exit status 1 on any mismatch.

    python scripts/fuzz_gpu.py --seconds 600 --seed 1

tests/test_gpu_fuzz.py runs a fixed number of cases of the same sweep (deterministic).
"""
import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import compare  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_1802_08557_b200 import _native, workloads  # noqa: E402

FORCE = [{}, {}, {}, {"BLP_CMULTI": "0"}, {"BLP_CONDENSED": "0"}, {"BLP_LAZY_SMALL": "0"}, {"BLP_LAZY": "0"},
         {"BLP_KERNEL": "smem"}, {"BLP_LAZY_SPLIT": "1"}, {"BLP_CT_STAGE": "2"}, {"BLP_CMULTI": "3"}]


def recipe(rng, m, n, cnt, seed):
    k = rng.integers(4)
    if k == 0 and m >= 2:
        A, b, c = workloads.afiro_arrays(cnt, seed=seed, m=m, n=n, infeasible_frac=float(rng.random() * 0.5))
    elif k == 1 and m >= 3 and n >= 5:
        A, b, c = workloads.degenerate_arrays(cnt, seed=seed, m=m, n=n)
    elif k == 2:
        A, b, c = workloads.random_arrays(max(m, n), cnt, seed)
        A, b, c = A[:, :m, :n], b[:, :m], c[:, :n]
    else:
        g = np.random.default_rng(seed)
        A = g.integers(-6, 7, size=(cnt, m, n)).astype(np.float64)
        b = g.integers(-4, 9, size=(cnt, m)).astype(np.float64)
        c = g.integers(-5, 6, size=(cnt, n)).astype(np.float64)
    return np.ascontiguousarray(A), np.ascontiguousarray(b), np.ascontiguousarray(c)


def run(seed: int, seconds: float | None = None, cases: int | None = None, log=print,
        huge: bool = False) -> tuple[int, int, int]:
    """Random cases until the time or case budget is spent; returns (cases, LPs, mismatches).
    huge: 400..700 rows/columns (the lazy, cluster and HBM-streamed families), single-phase
    random LPs and the degenerate recipe only (two-phase LPs of that size take the oracle
    minutes)."""
    rng = np.random.default_rng(seed)
    t_end = time.time() + seconds if seconds is not None else None
    done = bad = lps = 0
    while (t_end is None or time.time() < t_end) and (cases is None or done < cases):
        big = rng.random() < 0.1
        if huge:
            m, n, cnt = int(rng.integers(400, 701)), int(rng.integers(400, 701)), int(rng.integers(1, 4))
        else:
            m = int(rng.integers(1, 300 if big else 140))
            n = int(rng.integers(1, 300 if big else 140))
            cnt = int(rng.integers(1, 8 if big else 120))
        seed_k = int(rng.integers(1 << 30))
        if huge:
            if rng.random() < 0.5:
                A, b, c = workloads.random_arrays(max(m, n), cnt, seed_k)
                A, b, c = (np.ascontiguousarray(v) for v in (A[:, :m, :n], b[:, :m], c[:, :n]))
            else:
                A, b, c = workloads.degenerate_arrays(cnt, seed=seed_k, m=m, n=n)
                b = np.abs(b)
        else:
            A, b, c = recipe(rng, m, n, cnt, seed_k)
        shared = rng.random() < 0.2
        if shared:
            A, b = A[0].copy(), b[0].copy()
        lim = {}
        if rng.random() < 0.3:
            lim = dict(max_iterations=int(rng.integers(1, 60)))
        if rng.random() < 0.15:
            lim["anti_cycling"] = False
        if rng.random() < 0.15:
            lim["degenerate_pivot_limit"] = int(rng.integers(0, 6))
        env = FORCE[int(rng.integers(len(FORCE)))]
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            got = _native.solve_host(A, b, c, _native.make_limits(**lim), shared_Ab=shared)
            variant = _native.kernel_variant(m, n, shared)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        want = oracle.solve_batch(A, b, c, shared_Ab=shared, threads=oracle.host_cores(), **lim)
        try:
            valid = got["status"] != 4     # phase-1 unbounded: the API raises, outputs unspecified
            sub = lambda d: {k: np.asarray(d[k])[valid] for k in ("status", "objective", "x", "it1", "it2")}  # noqa: E731
            compare(sub(got), sub(want), "")
            assert np.array_equal(got["status"] == 4, want["status"] == 4)
        except AssertionError as e:
            bad += 1
            log(f"MISMATCH {m}x{n} cnt={cnt} seed={seed_k} shared={shared} lim={lim} env={env} {variant}: {e}")
        done += 1
        lps += cnt
    return done, lps, bad


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("--seconds", type=float, default=300)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--huge", action="store_true", help="400..700-sized single-phase / degenerate LPs")
    a = p.parse_args()
    cases, lps, bad = run(a.seed, seconds=a.seconds, log=lambda s: print(s, flush=True), huge=a.huge)
    print(f"fuzz: {cases} cases, {lps} LPs, {bad} mismatches", flush=True)
    sys.exit(1 if bad else 0)
