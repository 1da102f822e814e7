#!/bin/bash
# compute-sanitizer over every kernel family (scripts/san_run.py cases); logs to gpurun_out/sanitize/.
# usage: scripts/sanitize.sh [case ...]   (default: all cases, racecheck + synccheck + memcheck)
mkdir -p gpurun_out/sanitize
cases=${@:-$(python -c "import sys; sys.path.insert(0,'scripts'); import san_run; print(' '.join(san_run.CASES))")}
for c in $cases; do
  for tool in memcheck racecheck synccheck; do
    log=gpurun_out/sanitize/${c}_${tool}.log
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/san_run.py $c > $log 2>&1
    echo "$c $tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|parity=' $log | tr '\n' ' ')"
  done
done
