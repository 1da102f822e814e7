#!/bin/bash
# One gpurun round: parity tests + kernel sweep on the named configs; logs under gpurun_out/.
# usage: scripts/gpu_check.sh "c2:100000" "c4:200000" ...
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.log
for spec in "$@"; do
  cfg=${spec%%:*}; cnt=${spec#*:}
  python scripts/sweep.py --config "$cfg" --count "$cnt" --env "" >> gpurun_out/sweep.log 2>&1
done
cut -c1-220 gpurun_out/sweep.log
