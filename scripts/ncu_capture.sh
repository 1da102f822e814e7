#!/bin/bash
# ncu captures of one config's dominant kernel: launch list over prof_run.py, then one
# `--set full` capture of the kernel matching $3 (regex).  usage: scripts/ncu_capture.sh c2 100000 condensed tag
cfg=$1; cnt=$2; kre=$3; tag=$4
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python scripts/prof_run.py --config $cfg --count $cnt --launches 2 > gpurun_out/${tag}_lb.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:$kre --launch-skip 1 --launch-count 1 \
    -o gpurun_out/${tag} -f python scripts/prof_run.py --config $cfg --count $cnt --launches 2 > gpurun_out/${tag}_ncu.log 2>&1
tail -2 gpurun_out/${tag}_ncu.log
