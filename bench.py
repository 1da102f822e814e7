"""Benchmark of the batched two-phase simplex (BASELINE.json metric: LPs solved/sec, fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one batched solve of the whole per-GPU batch.  The default workload
is BASELINE.json configs[1] (C2): 1e5 afiro-shaped 28x32 LPs with mixed-sign
b (two-phase), per GPU (weak scaling: every rank solves its own 1e5 LPs,
contiguous LP-index shards of an N x 1e5 global batch, no collective on the
data path).  Rank 0 prints one JSON line:

  value      LPs/s over all ranks, inputs resident in HBM (blp_solve_batch_device),
             CUDA events on the launching stream, max over ranks
  e2e        same metric through the public API (batch_solve_arrays) from pinned
             host buffers: H2D of A, b, c + kernels + D2H of every result per step
  roofline   the dominant kernel's algorithmic bytes (or flops) / kernel time against
             the measured peak of the resource that bounds it (roofline_line)
  cpu_baseline  the C oracle port (oracle/, the reference algorithm) on the
             host cores, rank 0 at N=1, on a bounded sample of the workload
  parity     the timed outputs against the oracle on that sample: status, x,
             iterations exactly, objective as a true relative error

``--impl reference`` times that CPU implementation alone (rank 0; other ranks
exit 0) on the same config and prints the reference arm's line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LPs solved/sec (batch 1e5, fp64)"
UNIT = "LPs/s"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "c4b", "c5b"])
    p.add_argument("--count", type=int, default=None, help="LPs per GPU (default: the config's size)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def workload(cfg: str, count: int | None, rank: int):
    """Packed inputs of this rank's shard: rank r solves LPs [r*B, (r+1)*B) of the global batch,
    generated with the config's recipe and seed + 1000*r (rank 0 = the canonical config)."""
    from paper_1802_08557_b200 import workloads
    spec = workloads.CONFIGS[cfg]
    cnt = spec["count"] if count is None else count
    if cfg == "c1":
        A, b, c = workloads.random_arrays(5, cnt, 0 + 1000 * rank)
        shared = False
    elif cfg == "c2":
        A, b, c = workloads.afiro_arrays(cnt, seed=2 + 1000 * rank)
        shared = False
    elif cfg == "c3":
        A, b, c = workloads.degenerate_arrays(cnt, seed=3 + 1000 * rank)
        shared = False
    elif cfg == "c4":
        A, b = workloads.support_polytope()
        c = workloads.support_directions(cnt, offset=rank * cnt)
        shared = True
    elif cfg == "c4b":
        A, b = workloads.support_polytope_two_phase()
        c = workloads.support_directions(cnt, offset=rank * cnt)
        shared = True
    elif cfg == "c5b":
        A, b, c = workloads.big_two_phase_arrays(cnt, seed=55 + 1000 * rank)
        shared = False
    else:
        A, b, c = workloads.random_arrays(500, cnt, 5 + 1000 * rank)
        shared = False
    return A, b, c, shared, spec


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.2)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------

def bytes_per_pivot(m: int, n: int) -> int:
    """Algorithmic tableau bytes per pivot: one read + one write of (m+1)(n+m+1) fp64 cells."""
    return 16 * (m + 1) * (n + m + 1)


def measured_hbm_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_record(cfg: str, variant: str):
    """The committed `ncu --set full` capture summary of this config's kernel
    (profiles/traffic.json, written by scripts/ncu_summary.py), or None."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    recs = [r for r in json.loads(p.read_text()) if r.get("config") == cfg and r.get("variant") == variant]
    return recs[-1] if recs else None


def ncu_traffic(cfg: str, variant: str, count: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel from the committed
    capture (per-LP traffic x LPs when the capture used a sub-batch of the workload), or None."""
    rec = ncu_record(cfg, variant)
    if rec is None:
        return None
    return rec["dram_bytes_per_launch"] / rec["lps_per_launch"] * count


def cpu_baseline(A, b, c, shared, target_s: float = 10.0) -> tuple[dict, dict]:
    """The oracle port (reference algorithm in C) on all host cores, bounded sample.
    Returns (cpu_baseline line, the oracle's outcomes on that sample -- the parity checker)."""
    from oracle import oracle
    cores = oracle.host_cores()
    probe = min(len(c), 2000)
    t0 = time.perf_counter()
    oracle.solve_batch(A if shared else A[:probe], b if shared else b[:probe], c[:probe], shared_Ab=shared,
                       threads=cores)
    rate = probe / max(1e-6, time.perf_counter() - t0)
    sample = int(min(len(c), max(probe, rate * target_s)))
    t0 = time.perf_counter()
    res = oracle.solve_batch(A if shared else A[:sample], b if shared else b[:sample], c[:sample],
                             shared_Ab=shared, threads=cores)
    dt = time.perf_counter() - t0
    line = {"value": sample / dt, "unit": UNIT, "cores": int(res["threads"]), "kind": "port",
            "sample": f"first {sample} LPs of this config's rank-0 batch, oracle/blp_oracle.c "
                      f"(full reference tableau incl. artificial columns), {res['threads']} threads, {dt:.2f} s",
            "pivots_per_s": float((res["it1"] + res["it2"]).sum() / dt)}
    return line, res


def parity(got: dict, want: dict) -> dict:
    """The timed GPU outputs against the oracle on the same LPs (the first len(want) of them):
    status, x and per-phase iterations exactly; objective as a true relative error."""
    k = len(want["status"])
    gs, ws = got["status"][:k], want["status"]
    opt = (gs == 0) & (ws == 0)
    x_bad = int((~(got["x"][:k][opt] == want["x"][opt]).all(axis=1)).sum()) if opt.any() else 0
    go, wo = got["objective"][:k][opt], want["objective"][opt]
    diff = np.abs(go - wo)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(diff == 0, 0.0, diff / np.abs(wo))
    return {"checked": int(k), "of": int(len(got["status"])), "status_mismatch": int((gs != ws).sum()),
            "x_mismatch": x_bad,
            "iter_mismatch": int(((got["it1"][:k] != want["it1"]) | (got["it2"][:k] != want["it2"])).sum()),
            "max_obj_rel": float(rel.max()) if rel.size else 0.0, "obj_rtol": 1e-9,
            "checker": "oracle/blp_oracle.c (C restatement of the reference, pinned to tests/golden/)"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    A, b, c, shared, spec = workload(args.config, args.count, 0)
    from oracle import oracle
    cores = oracle.host_cores()
    # size one step at ~2 s of host work so warmup+steps finish in a few minutes
    probe = min(len(c), 2000)
    t0 = time.perf_counter()
    oracle.solve_batch(A if shared else A[:probe], b if shared else b[:probe], c[:probe], shared_Ab=shared,
                       threads=cores)
    rate = probe / max(1e-6, time.perf_counter() - t0)
    sample = int(min(len(c), max(probe, rate * 2.0)))
    sl = (lambda v: v) if shared else (lambda v: v[:sample])
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = oracle.solve_batch(sl(A), sl(b), c[:sample], shared_Ab=shared, threads=cores)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    step = statistics.median(times)
    value = sample / step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(args, spec, len(c), shared),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": int(res["threads"]), "kind": "port",
                         "sample": f"first {sample} LPs of the rank-0 batch per step, oracle/blp_oracle.c "
                                   f"(C restatement of batchlp tableau.py/simplex.py), median of {args.steps} steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "pivots_per_s": float((res["it1"] + res["it2"]).sum() / step),
    }
    print(json.dumps(line), flush=True)


def config_block(args, spec, count, shared) -> dict:
    from paper_1802_08557_b200 import workloads
    m, n = spec["m"], spec["n"]
    return {"workload": f"{args.config}: {spec['doc']}", "m": m, "n": n, "lps_per_gpu": count,
            "global_batch": count * args.gpus, "support_function": shared,
            "parallelism": f"lp-index shards x{args.gpus} (no collective)",
            "l2": "inputs > 126 MB L2 per step (no flush needed)" if count * (m * n + m + n) * 8 > 126e6
            else "inputs fit L2; L2 flushed between steps"}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_1802_08557_b200 import SolverLimits, _native, batch_solve_arrays

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # One process per GPU.  BLP_BENCH_SHARE_GPU=1 folds ranks onto the visible GPUs and uses
    # gloo for the scalar collectives: a functional check of the multi-rank path on a 1-GPU box.
    share = os.environ.get("BLP_BENCH_SHARE_GPU") == "1"
    local_dev = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    A, b, c, shared, spec = workload(args.config, args.count, rank)
    count, n = c.shape
    m = b.shape[-1]
    lim = SolverLimits().to_native()
    tA, tb, tc = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (A, b, c))
    out = dict(status=torch.empty(count, dtype=torch.int8, device=dev),
               objective=torch.empty(count, dtype=torch.float64, device=dev),
               x=torch.empty(count, n, dtype=torch.float64, device=dev),
               it1=torch.empty(count, dtype=torch.int32, device=dev),
               it2=torch.empty(count, dtype=torch.int32, device=dev))
    stream = torch.cuda.current_stream(dev)
    l2_flush = None
    inputs_bytes = count * (m * n + m + n) * 8 if not shared else (m * n + m + count * n) * 8
    if inputs_bytes <= 256e6:
        l2_flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=dev)

    def step():
        if l2_flush is not None:
            l2_flush.zero_()
        _native.solve_device(tA, tb, tc, lim, out, shared_Ab=shared, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
        step()
    barrier()

    # ---- device-resident value: CUDA events per step on the launching stream ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = _native.launch_count()
    with ClockSampler(local_dev) as clocks:
        barrier()
        t_all0 = torch.cuda.Event(enable_timing=True)
        t_all1 = torch.cuda.Event(enable_timing=True)
        t_all0.record(stream)
        for e0, e1 in evs:
            if l2_flush is not None:
                l2_flush.zero_()
            e0.record(stream)
            _native.solve_device(tA, tb, tc, lim, out, shared_Ab=shared, stream=stream)
            e1.record(stream)
        t_all1.record(stream)
        barrier()
    launches = _native.launch_count() - launches0
    kernel_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    step_ms = statistics.mean(kernel_ms)
    region_ms = t_all0.elapsed_time(t_all1)
    res = {k: v.cpu().numpy() for k, v in out.items()}
    pivots = int((res["it1"].astype(np.int64) + res["it2"]).sum())

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device='cpu' if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device='cpu' if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    ms_per_step = max_over_ranks(step_ms)
    total_lps = count * world
    value = total_lps / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel ----
    variant = _native.kernel_variant(m, n, shared)
    secs = step_ms / 1e3
    if variant.startswith("lazy+"):
        # the lazy tableau hands phase-1 LPs (b < 0) and LPs past its pivot budget to the dense
        # family in the same launch sequence; when it keeps under half of the batch, the dense
        # kernel dominates the step and its roofline is the one that applies (C3: every LP)
        two_phase = np.broadcast_to(np.any(b < 0, axis=-1), (count,))
        deferred = float(np.mean(two_phase | ((res["it1"] + res["it2"]) > 64)))
        if deferred > 0.5:
            variant = variant[len("lazy+"):]
    input_bytes = (A.nbytes if not shared else 0) + (b.nbytes if not shared else 0) + c.nbytes
    output_bytes = count * (1 + 8 + 8 * n + 4 + 4)
    roofline = roofline_line(variant, m, n, pivots, secs, input_bytes, output_bytes,
                             smem_peak=_native.probe_smem_gbs(local_dev),
                             fp64_peak=_native.probe_fp64_gflops(local_dev) / 1e3,
                             traffic=ncu_traffic(args.config, variant, count))
    rec = ncu_record(args.config, variant)
    if rec is not None:
        # what the committed capture says binds the kernel (pipe utilisations, 0..1)
        roofline["ncu"] = {k: rec.get(k) for k in ("issue_active", "fp64_pipe", "smem_pipe")} | \
                          {"source": rec.get("source")}

    # ---- e2e through the public API from pinned host buffers, on this rank's GPU ----
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    hA, hb, hc = pin(A), pin(b), pin(c)
    h2d = hA.nbytes + hb.nbytes + hc.nbytes
    d2h = count * (1 + 8 + 8 * n + 4 + 4)
    from paper_1802_08557_b200 import support_batch
    devs = (local_dev,)
    call = (lambda: support_batch(hA, hb, hc, devices=devs)) if shared else \
        (lambda: batch_solve_arrays(hA, hb, hc, devices=devs))
    call()
    barrier()
    e2e_t = []
    for _ in range(max(3, min(args.steps, 10))):
        barrier()
        t0 = time.perf_counter()
        r = call()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(statistics.median(e2e_t))
    torch.cuda.set_device(local_dev)
    h2d_gbs = pinned_h2d_gbs(torch, dev)
    assert np.array_equal(r.status, res["status"]) and np.array_equal(r.x, res["x"]), "e2e result differs"

    obj_api = object_api_e2e(A, b, c, shared, local_dev, res, barrier, max_over_ranks, world, args)

    total_pivots = sum_over_ranks(pivots)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (workloads recipe, seed+1000*rank)",
        "config": config_block(args, spec, count, shared) | {"kernel": variant},
        "pivots_per_s": total_pivots / (ms_per_step / 1e3),
        "status_counts": {str(k): int(v) for k, v in zip(*np.unique(res["status"], return_counts=True))},
        "roofline": roofline,
        "e2e": {"value": total_lps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3,
                "h2d_pinned_gbs": h2d_gbs, "h2d_floor_ms": h2d / h2d_gbs / 1e6,
                "api": "batch_solve_arrays / support_batch (blp_solve_batch_host: sub-batches pipelined "
                       "over 4 streams)"},
        "e2e_object_api": obj_api,
        "gpu_launches": int(launches),
        "timed_region_ms": region_ms,
        "clocks": clocks.summary(),
    }
    # ---- parity of the timed outputs against the oracle (after timing) ----
    if world == 1:
        if rank == 0 and not args.no_cpu_baseline:
            base, want = cpu_baseline(A, b, c, shared)
            line["cpu_baseline"] = base
            line["parity"] = parity(res, want)
    else:
        # every rank checks a bounded prefix of its own shard; mismatch counts summed over ranks
        from oracle import oracle
        k = min(count, 5000)
        want = oracle.solve_batch(A if shared else A[:k], b if shared else b[:k], c[:k], shared_Ab=shared,
                                  threads=max(1, oracle.host_cores() // world))
        pr = parity(res, want)
        for key in ("checked", "of", "status_mismatch", "x_mismatch", "iter_mismatch"):
            pr[key] = int(sum_over_ranks(pr[key]))
        pr["max_obj_rel"] = max_over_ranks(pr["max_obj_rel"])
        line["parity"] = pr
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def object_api_e2e(A, b, c, shared, dev: int, res: dict, barrier, max_over_ranks, world: int, args) -> dict:
    """The reference-facing call itself: batch_solve(list[StandardFormLP], BatchConfig) on
    this rank's batch (batch.py:134-179), wall clock per call with the list built beforehand
    (as the reference bench does, cli.py:316-318).  host_marshalling_ms = the C pass over
    the list (_pyobj.collect) -- the rest of the call is the pipelined gather + H2D +
    kernels + D2H inside the library, and the lazy outcome list."""
    from paper_1802_08557_b200 import BatchConfig, StandardFormLP, _pyobj, batch_solve
    from paper_1802_08557_b200.model import STATUS_BY_CODE
    count = len(c)
    lps = [StandardFormLP(c=c[k], A=A if shared else A[k], b=b if shared else b[k]) for k in range(count)]
    cfg = BatchConfig(devices=(dev,))
    rep = batch_solve(lps, cfg)
    times, collect = [], []
    for _ in range(max(3, min(args.steps, 5))):
        barrier()
        t0 = time.perf_counter()
        _pyobj.collect(lps, b.shape[-1], c.shape[1])
        collect.append(time.perf_counter() - t0)
        barrier()
        t0 = time.perf_counter()
        rep = batch_solve(lps, cfg)
        times.append(time.perf_counter() - t0)
    wall = max_over_ranks(statistics.median(times))
    want = {STATUS_BY_CODE[int(k)].value: int(v) for k, v in zip(*np.unique(res["status"], return_counts=True))}
    assert rep.status_counts() == want, "object API result differs"
    k = int(np.argmax(res["status"] == 0)) if (res["status"] == 0).any() else 0
    o = rep.outcomes[k]                                   # spot-check one materialised outcome
    assert o.iterations_phase2 == int(res["it2"][k]) and (o.primal_point is None or
                                                          np.array_equal(o.primal_point, res["x"][k]))
    return {"value": count * world / wall, "unit": UNIT, "ms_per_call": wall * 1e3,
            "host_marshalling_ms": statistics.median(collect) * 1e3, "chunks": rep.plan.count,
            "api": "batch_solve(list[StandardFormLP], BatchConfig) -> BatchReport "
                   "(_pyobj.collect + blp_solve_batch_gather; outcomes built on access)"}


def pinned_h2d_gbs(torch, dev, nbytes: int = 512 << 20) -> float:
    """Pinned host -> device copy rate on a 512 MB buffer (events on an explicit stream of `dev`):
    the PCIe floor the e2e number is compared with."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(device=dev)
    best = 0.0
    with torch.cuda.stream(s):
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            d.copy_(h, non_blocking=True)
            e1.record(s)
            s.synchronize()
            best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def roofline_line(variant: str, m: int, n: int, pivots: int, secs: float, input_bytes: int, output_bytes: int,
                  *, smem_peak: float, fp64_peak: float, traffic) -> dict:
    """Roofline of the dominant kernel, with `achieved` always a physical rate of the bound
    resource (so frac <= 1 up to measurement noise):

    * dense on-chip tableaux (warplp*, pairlp/quadlp, regtile, smem_rpl*, cluster_r*):
      SURVEY.md §8(d)'s 16(m+1)(n+m+1) B per pivot -- every cell read and written once --
      against the measured shared-memory bandwidth; FP64 view alongside;
    * HBM-streamed tableaux (hbm_rpl*): the same bytes against the measured HBM rate;
    * the exact lazy tableau (lazy+*): the dense tableau is never materialised, so the
      kernel's algorithmic floor is one HBM read of the inputs plus the outputs, against the
      measured HBM rate; `dense_equiv_gbs` keeps the §8(d) figure for comparison only.
    """
    hbm_peak, hbm_src = measured_hbm_gbs()
    smem_src = "measured in-run (blp_probe_smem_gbs: LDS.128+STS.128, all SMs)"
    dense_bpp = bytes_per_pivot(m, n)
    dense_gbs = pivots * dense_bpp / secs / 1e9
    fpp = 2 * (m + 1) * (n + m + 1)
    base = {"kernel": variant, "pivots_per_launch": pivots, "dense_bytes_per_pivot": dense_bpp,
            "hbm_peak_gbs": hbm_peak, "smem_peak_gbs": smem_peak, "fp64_peak_tflops": fp64_peak}
    if variant.startswith("lazy"):
        io = input_bytes + output_bytes
        achieved = io / secs / 1e9
        line = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic, "peak_source": hbm_src, "algorithmic_bytes_per_launch": io,
                "algorithmic": "inputs read once + outputs written once (the lazy tableau's floor)",
                "dense_equiv_gbs": dense_gbs}
        if traffic:
            line["traffic_over_algorithmic"] = traffic / io
    elif variant.startswith(("ctab", "cm")):
        # condensed tableau (blp_condensed_kernel.cuh, blp_cmulti_kernel.cuh): only the
        # (m+1) x (n+1) nonbasic + rhs cells exist, in registers (cm*: a few slots per row in a
        # shared tile) -- the physical resource the update consumes is the FP64 pipe: one
        # DMUL + one DADD per cell
        cfp = 2 * (m + 1) * (n + 1)
        fl = pivots * cfp / secs / 1e12
        line = {"bound": "fp64", "achieved": fl, "peak": fp64_peak, "unit": "TFLOP/s", "frac": fl / fp64_peak,
                "traffic": traffic, "peak_source": "measured in-run (blp_probe_fp64_gflops: unfused DMUL+DADD, "
                                                   "all SMs)",
                "flops_per_pivot": cfp,
                "algorithmic": "2 flops per condensed-tableau cell per pivot ((m+1)(n+1) cells, registers)",
                "dense_equiv_gbs": dense_gbs, "dense_equiv_smem_frac": dense_gbs / smem_peak}
        if traffic:
            line["traffic_over_io"] = traffic / (input_bytes + output_bytes)
    elif variant.startswith("hbm"):
        line = {"bound": "hbm", "achieved": dense_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": dense_gbs / hbm_peak, "traffic": traffic, "peak_source": hbm_src,
                "bytes_per_pivot": dense_bpp}
    else:
        line = {"bound": "smem", "achieved": dense_gbs, "peak": smem_peak, "unit": "GB/s",
                "frac": dense_gbs / smem_peak, "traffic": traffic, "peak_source": smem_src,
                "bytes_per_pivot": dense_bpp,
                "fp64_achieved_tflops": pivots * fpp / secs / 1e12,
                "fp64_frac": pivots * fpp / secs / 1e12 / fp64_peak}
    return base | line


if __name__ == "__main__":
    main()
