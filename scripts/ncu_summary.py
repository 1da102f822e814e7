"""Summarise an `ncu --set full` capture into profiles/: key metrics of the captured kernel
and its DRAM traffic per launch (bench.py's roofline.traffic reads profiles/traffic.json).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep --config c2 --lps 100000 --out profiles/r01_c2_full.txt
"""
import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__shared_mem_per_block_dynamic")

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--config", required=True)
ap.add_argument("--lps", type=int, required=True)
ap.add_argument("--variant", default=None, help="blp_kernel_variant name (bench.py looks traffic up by it)")
ap.add_argument("--out", required=True)
ap.add_argument("--traffic", default="profiles/traffic.json", help="traffic table to update")
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
lines = []
traffic = []
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "?")
    lines.append(f"kernel: {name}")
    for k in KEYS:
        if k in d:
            lines.append(f"  {k} = {d[k]} {u.get(k, '')}")
    rb = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
    wb = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rb *= scale.get(u.get("dram__bytes_read.sum", "byte"), 1)
    wb *= scale.get(u.get("dram__bytes_write.sum", "byte"), 1)
    lines.append(f"  dram bytes per launch = {rb + wb:.0f}")
    pct = lambda k: round(float(d[k].replace(",", "")) / 100, 4) if d.get(k) else None  # noqa: E731
    traffic.append(dict(kernel=name, dram_bytes_per_launch=rb + wb,
                        issue_active=pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                        fp64_pipe=pct("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                        smem_pipe=pct("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")))
Path(a.out).write_text("\n".join(lines) + "\n")
print("\n".join(lines))
variant = None
for t in traffic:
    k = t["kernel"]
    if "warplp_kernel<64" in k:
        variant = "warplp_c64"
    elif "warplp_kernel<32" in k:
        variant = "warplp_c32"
    elif "regtile" in k:
        variant = "regtile"
    elif "tableau_kernel" in k:
        variant = ("smem" if "(bool)1" in k else "hbm")
    t["variant_family"] = a.variant or variant
tj = Path(a.traffic)
recs = json.loads(tj.read_text()) if tj.exists() else []
for t in traffic:
    # one record per (config, LPs, variant): bench.py looks traffic up by variant
    recs = [r for r in recs if not (r["config"] == a.config and r["lps_per_launch"] == a.lps
                                    and (r["kernel"] == t["kernel"] or r["variant"] == t["variant_family"]))]
    recs.append(dict(config=a.config, lps_per_launch=a.lps, kernel=t["kernel"], variant=t["variant_family"],
                     dram_bytes_per_launch=t["dram_bytes_per_launch"], issue_active=t["issue_active"],
                     fp64_pipe=t["fp64_pipe"], smem_pipe=t["smem_pipe"], source=a.out))
tj.write_text(json.dumps(recs, indent=1) + "\n")
