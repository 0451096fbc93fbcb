#!/bin/bash
# one-launch step experiments: optional parity subset, then bench ms_per_step per setting
# usage: SETTINGS="EPFEM_MEGA=0 EPFEM_MEGA_SLACK=0,EPFEM_MEGA_KB=20" (space-separated runs, comma-separated vars)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -x -q -m gpu -k "cfg2 or MEGA" > gpurun_out/pytest_mega.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mega.log
fi
for s in ${SETTINGS:-default}; do
X
  env $vars timeout 300 python bench.py --config ${CFG:-cfg2} --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/mega_$s.json 2>gpurun_out/mega_$s.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/mega_$s.json').read().strip().splitlines()[-1]); print('$s', round(d['ms_per_step'],4), d['kernels_ms'])" >> gpurun_out/mega_summary.txt 2>&1
done
