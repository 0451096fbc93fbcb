#!/bin/bash
# BASELINE configs 4 / 5 plastic-fraction sweeps (one GPU, under gpurun):
# cfg4 at 0 / 25 / 50 / 100 %, cfg5 at 0 / 50 / 100 % -> gpurun_out/plastic_<cfg>_<frac>.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in 0 0.25 0.5 1.0; do
  timeout 900 python bench.py --config cfg4 --target $t --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/plastic_cfg4_$t.json 2> gpurun_out/plastic_cfg4_$t.err
done
for t in 0 0.5 1.0; do
  timeout 900 python bench.py --config cfg5 --target $t --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/plastic_cfg5_$t.json 2> gpurun_out/plastic_cfg5_$t.err
done
