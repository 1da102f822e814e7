#!/bin/bash
# One gpurun call: GPU test suite, every config's bench line, then (NCU=1) ncu captures of each
# config's dominant kernel: launch list + one --set full capture, summarised on the box
# (gpurun_out/profiles/, gpurun_out/traffic.json) and the .ncu-rep dropped unless KEEP_REP=1
# (gpurun copies back at most 64 MiB).
mkdir -p gpurun_out/profiles
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/smi.txt 2>&1
free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
  tail -5 gpurun_out/pytest_gpu.log
fi
[ -z "$SKIP_BENCH" ] && bash scripts/bench_all.sh
if [ -n "$NCU" ]; then
  cp profiles/traffic.json gpurun_out/traffic.json
  for spec in "c2 100000 condensed r02_c2_ctab" "c3 20000 cmulti r02_c3_cm4" "c4 1000000 cmulti r02_c4_cm2" \
              "c5 10000 lazy_kernel r02_c5_lazy"; do
    set -- $spec
    bash scripts/ncu_capture.sh $1 $2 $3 $4
    variant=$(python -c "import sys; sys.path.insert(0, '.'); import bench; from paper_1802_08557_b200 import _native; \
A, b, c, sh, _ = bench.workload('$1', 8, 0); print(_native.kernel_variant(b.shape[-1], c.shape[1], sh))")
    python scripts/launch_summary.py gpurun_out/$4_launches.csv > gpurun_out/profiles/$(echo $4 | cut -d_ -f1-2)_launches.txt
    python scripts/ncu_summary.py gpurun_out/$4.ncu-rep --config $1 --lps $2 --variant "$variant" \
        --out gpurun_out/profiles/$4_full.txt --traffic gpurun_out/traffic.json > /dev/null
    ncu -i gpurun_out/$4.ncu-rep --page source --csv --print-source=sass > gpurun_out/profiles/$4_sass.csv 2>/dev/null
    gzip -f gpurun_out/profiles/$4_sass.csv
    [ -z "$KEEP_REP" ] && rm -f gpurun_out/$4.ncu-rep
  done
fi
