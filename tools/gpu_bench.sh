#!/bin/bash
# One GPU session: the default bench line (driver command) and the reference
# arm, with wall times (writes gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
s=$(date +%s)
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$? wall=$(( $(date +%s) - s ))" >> gpurun_out/bench_rc.txt
if [ -z "$NO_REF" ]; then
s=$(date +%s)
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference rc=$? wall=$(( $(date +%s) - s ))" >> gpurun_out/bench_rc.txt
fi
