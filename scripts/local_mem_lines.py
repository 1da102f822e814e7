"""Which source lines of a kernel touch local memory (STL/LDL) -- register-array demotion finder.

    python scripts/local_mem_lines.py <kernel-substring>
"""
import re
import subprocess
import sys
from collections import Counter

sub = sys.argv[1]
subprocess.run(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                "-fmad=false", "-cubin", "-o", "/tmp/blp_lm.cubin",
                "paper_1802_08557_b200/csrc/blp_capi.cu"], check=True)
txt = subprocess.run(["nvdisasm", "-g", "/tmp/blp_lm.cubin"], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(txt) if l.startswith(".text.") and sub in l)
cur, cnt = None, Counter()
for l in txt[start + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    if re.search(r"\b(STL|LDL)", l):
        cnt[cur] += 1
for k, v in cnt.most_common(20):
    print(v, k)
