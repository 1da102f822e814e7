"""Summarise an ncu report's source page: hottest CUDA source lines by warp-stall samples,
with executed warp instructions per line (needs -lineinfo).

    python scripts/ncu_hot.py gpurun_out/prof.ncu-rep [--top 40]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
lines = []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        stall, inst = int(r[4] or 0), int(r[7] or 0)
    except (ValueError, IndexError):
        continue
    lines.append((stall, inst, f"{fname}:{r[0]}", r[1].strip()))
ts = sum(s for s, *_ in lines) or 1
ti = sum(i for _, i, *_ in lines) or 1
print(f"stall samples {ts}, warp instructions {ti}")
print(" stall%  inst%   location                      source")
for s, i, loc, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/ts:6.1f} {100*i/ti:6.1f}   {loc:28s} {src[:80]}")
