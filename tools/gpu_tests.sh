#!/bin/bash
# One GPU session: the -m gpu suite with per-test durations, smoke (writes gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
s=$(date +%s)
EPFEM_PARITY_LOG=gpurun_out/parity.jsonl timeout ${PYT_TIMEOUT:-2400} python -m pytest tests -x -q -m gpu --durations=25 ${PYT_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$? wall=$(( $(date +%s) - s ))" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
