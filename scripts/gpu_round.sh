#!/bin/bash
# One gpurun call: GPU test suite, every config's bench line, then ncu captures of each config's
# dominant kernel (launch list + one --set full capture; summaries via scripts/ncu_summary.py).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/smi.txt 2>&1
free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
bash scripts/bench_all.sh
if [ -n "$NCU" ]; then
  bash scripts/ncu_capture.sh c2 100000 condensed r02_c2_ctab
  bash scripts/ncu_capture.sh c3 20000 cmulti r02_c3_cm4
  bash scripts/ncu_capture.sh c4 1000000 cmulti r02_c4_cm2
  bash scripts/ncu_capture.sh c5 10000 lazy_kernel r02_c5_lazy
fi
