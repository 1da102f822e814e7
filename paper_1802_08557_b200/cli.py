"""``bench`` timing surface with GPU rows.

    python -m paper_1802_08557_b200 bench [--dims 5,28,50,100] [--batch-sizes 100,1000,10000,100000]

Emits the reference's bench CSV (/root/reference/pkg/src/batchlp/cli.py:42-46,
304-333) column for column -- ``dim,batch_size,repeats,setup_ms,wall_ms,
lps_per_sec,n_optimal,n_unbounded,n_infeasible,n_iteration_limit`` -- over the
same sweep (``gen_random_lps(dim, size, seed + cell)``, setup = workload
generation, wall = mean ``batch_solve`` total over the repeats), so the
paper-style sweep is reported directly, here with the batch solved on the GPU.
``--extended`` appends the GPU columns (kernel variant, pivots/s, packed-array
wall time with the object layers skipped).  Flags fall back to BATCHLP_*
environment variables as in the reference (cli.py:48-55); the other reference
subcommands (solve / batch / gen / verify) are outside the batched path.
"""
from __future__ import annotations

import argparse
import csv
import os
import sys
import time

import numpy as np

BENCH_DIMS = (5, 28, 50, 100)
BENCH_BATCH_SIZES = (100, 1_000, 10_000, 100_000)
BENCH_CSV_HEADER = ("dim", "batch_size", "repeats", "setup_ms", "wall_ms", "lps_per_sec", "n_optimal",
                    "n_unbounded", "n_infeasible", "n_iteration_limit")
EXTENDED_HEADER = ("kernel", "pivots_per_lp", "arrays_wall_ms", "arrays_lps_per_sec")
ENV_PREFIX = "BATCHLP_"


def _env(flag: str, cast, fallback):
    raw = os.environ.get(ENV_PREFIX + flag.upper().replace("-", "_"))
    if raw is None:
        return fallback
    if cast is bool:
        return raw.strip().lower() in ("1", "true", "yes", "on")
    return cast(raw)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_1802_08557_b200",
                                     description="Batched dense LP solving on B200 (bench surface).")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bench", help="timing sweep over dims and batch sizes (CSV)")
    p.add_argument("--dim", type=int, default=_env("dim", int, None), help="(accepted for compatibility)")
    p.add_argument("--count", type=int, default=_env("count", int, None),
                   help="limit the number of sweep cells (0 = header only)")
    p.add_argument("--seed", type=int, default=_env("seed", int, 0))
    p.add_argument("--feasible-start", action=argparse.BooleanOptionalAction,
                   default=_env("feasible-start", bool, True))
    p.add_argument("--workers", type=int, default=_env("workers", int, 1))
    p.add_argument("--memory-budget", type=int, default=_env("memory-budget", int, 1 << 30))
    p.add_argument("--limits-max-iters", type=int, default=_env("limits-max-iters", int, None))
    p.add_argument("--repeats", type=int, default=_env("repeats", int, 10))
    p.add_argument("--dims", default=_env("dims", str, None))
    p.add_argument("--batch-sizes", default=_env("batch-sizes", str, None))
    p.add_argument("--devices", default=_env("devices", str, "0"), help="comma-separated CUDA devices")
    p.add_argument("--extended", action="store_true", help="append the GPU columns")
    p.set_defaults(func=cmd_bench)
    return parser


def cmd_bench(args) -> int:
    from . import BatchConfig, SolverLimits, _native, batch_solve, batch_solve_arrays, gen_random_lps
    from .workloads import random_arrays

    dims = [int(v) for v in args.dims.split(",")] if args.dims else list(BENCH_DIMS)
    sizes = [int(v) for v in args.batch_sizes.split(",")] if args.batch_sizes else list(BENCH_BATCH_SIZES)
    cells = [(d, s) for d in dims for s in sizes]
    if args.count is not None:
        cells = cells[:max(args.count, 0)]
    out = csv.writer(sys.stdout, lineterminator="\n")
    out.writerow(BENCH_CSV_HEADER + (EXTENDED_HEADER if args.extended else ()))
    devices = tuple(int(v) for v in str(args.devices).split(","))
    limits = SolverLimits(max_iterations=args.limits_max_iters)
    config = BatchConfig(memory_budget_bytes=args.memory_budget, worker_count=args.workers, limits=limits,
                         devices=devices)
    repeats = max(args.repeats, 1)
    for cell, (dim, size) in enumerate(cells):
        t0 = time.perf_counter()
        lps = gen_random_lps(dim, size, args.seed + cell, args.feasible_start)
        setup_s = time.perf_counter() - t0
        walls, report = [], None
        for _ in range(repeats):
            report = batch_solve(lps, config)
            walls.append(report.total_seconds)
        counts = report.status_counts()
        wall = sum(walls) / len(walls)
        row = [dim, size, repeats, f"{setup_s * 1e3:.3f}", f"{wall * 1e3:.3f}",
               f"{size / wall:.3f}" if wall > 0 else "inf",
               counts.get("optimal", 0), counts.get("unbounded", 0), counts.get("infeasible", 0),
               counts.get("iteration_limit", 0)]
        if args.extended:
            A, b, c = random_arrays(dim, size, args.seed + cell, args.feasible_start)
            res = batch_solve_arrays(A, b, c, limits, devices=devices)
            t1 = time.perf_counter()
            for _ in range(repeats):
                res = batch_solve_arrays(A, b, c, limits, devices=devices)
            aw = (time.perf_counter() - t1) / repeats
            piv = float(np.mean(res.iterations_phase1.astype(np.int64) + res.iterations_phase2)) if size else 0.0
            row += [_native.kernel_variant(dim, dim), f"{piv:.3f}", f"{aw * 1e3:.3f}",
                    f"{size / aw:.3f}" if aw > 0 else "inf"]
        out.writerow(row)
        sys.stdout.flush()
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (OSError, ValueError) as err:
        print(f"error: {err}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
