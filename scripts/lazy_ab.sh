#!/bin/bash
# Labelled A/B of libblp variants on the lazy-path workloads: C5 (1e4), C4 (1e6), random 100x100 (2e4).
#   scripts/lazy_ab.sh libblp_h0.so libblp_h1.so ...
for lib in "$@"; do
  c5=$(BLP_LIBRARY=$PWD/paper_1802_08557_b200/$lib python scripts/sweep.py --config c5 --count 10000 2>&1 | python -c "import sys,json; print(round(json.loads(sys.stdin.read().strip().splitlines()[-1])['ms'],3))")
  c4=$(BLP_LIBRARY=$PWD/paper_1802_08557_b200/$lib python scripts/sweep.py --config c4 --count 1000000 2>&1 | python -c "import sys,json; print(round(json.loads(sys.stdin.read().strip().splitlines()[-1])['ms'],3))")
  d1=$(BLP_LIBRARY=$PWD/paper_1802_08557_b200/$lib python scripts/lazy_vs_dense.py --dims 100 --count 20000 2>&1 | python -c "import sys,json; print(round(json.loads(sys.stdin.read().strip().splitlines()[-1])['lazy_ms'],3))")
  echo "$lib c5=$c5 c4=$c4 d100=$d1"
done
