#!/bin/bash
# Source-level stall profile of the standalone element-delta kernel (or K=regex) on cfg4 at a plastic
# fraction (under gpurun): T=1.0 K=k_elem_delta_staged bash tools/prof_delta.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${T:-1.0}; KR=${K:-k_elem_delta_staged}; C=${CFG:-cfg4}; TAG=${TAG:-delta}
CMD="python tools/time_paths.py --target=$T $C"
$CMD > gpurun_out/prof_${TAG}_plain.log 2>&1 || exit 1
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none -k regex:"$KR" -s 3 -c 1 -o /tmp/src_prof -f $CMD > gpurun_out/prof_${TAG}_ncu.log 2>&1
$NCU -i /tmp/src_prof.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${TAG}_sass.csv 2>&1
$NCU -i /tmp/src_prof.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>&1
gzip -f gpurun_out/prof_${TAG}_*.csv
