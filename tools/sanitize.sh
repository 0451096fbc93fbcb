#!/bin/bash
# compute-sanitizer racecheck / memcheck / synccheck of the hot kernels on small
# cfg2 / cfg4 / cfg5 meshes (under gpurun; writes gpurun_out/sanitize_*.log)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck memcheck synccheck; do
  for c in "cfg2 12" "cfg4 6" "cfg5 3" "cfg3 4"; do
    set -- $c
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_step.py $1 $2 \
      > gpurun_out/sanitize_${tool}_$1.log 2>&1
    echo "$tool $1 rc=$?" >> gpurun_out/sanitize_rc.txt
  done
done
