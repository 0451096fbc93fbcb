#!/bin/bash
# Source-level stall profile of one kernel (under gpurun): K=regex CFG=cfg2 bash tools/prof_source.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C=${CFG:-cfg2}; KR=${K:-k_newton_warp}
CMD="python bench.py --config $C --steps 2 --warmup 3 --no-cpu --no-e2e --no-side --extra none"
$CMD > /dev/null 2>&1 || exit 1
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none -k regex:"$KR" -s 1 -c 1 -o /tmp/src_prof -f $CMD > gpurun_out/src_ncu.log 2>&1
$NCU -i /tmp/src_prof.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${C}_sass.csv 2>&1
$NCU -i /tmp/src_prof.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${C}_cuda.csv 2>&1
$NCU -i /tmp/src_prof.ncu-rep --page raw --csv > gpurun_out/src_${C}_raw.csv 2>&1
gzip -f gpurun_out/src_${C}_*.csv
