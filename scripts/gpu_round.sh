#!/bin/bash
# One gpurun call: GPU test suite, then every config's bench line (logs under gpurun_out/).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/smi.txt 2>&1
free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
bash scripts/bench_all.sh
