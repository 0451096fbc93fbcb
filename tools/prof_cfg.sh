#!/bin/bash
# ncu evidence for one config (run under gpurun, one GPU): the bench command
# first without ncu, then the launch list (--metrics, every launch) and one
# --set full capture of the two hot kernels.  usage: CFG=cfg4 bash tools/prof_cfg.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C=${CFG:-cfg2}
CMD="python bench.py --config $C --steps 2 --warmup 3 --no-cpu --no-e2e --no-side --extra none"
$CMD > gpurun_out/prof_${C}_bench.json 2> gpurun_out/prof_${C}_bench.err || exit 1
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none -c ${NLAUNCH:-400} --csv --log-file gpurun_out/${C}_launches.csv $CMD > gpurun_out/prof_${C}_ncu1.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"${KR:-k_newton|k_row_stream}" -s ${SKIP:-2} -c ${COUNT:-2} \
  -o /tmp/${C}_prof -f $CMD > gpurun_out/prof_${C}_ncu2.log 2>&1
# the .ncu-rep stays on the box (size); its raw page and source hot spots come back
$NCU -i /tmp/${C}_prof.ncu-rep --page raw --csv > gpurun_out/${C}_raw.csv 2>&1
$NCU -i /tmp/${C}_prof.ncu-rep --page details --csv > gpurun_out/${C}_details.csv 2>&1
gzip -f gpurun_out/${C}_launches.csv gpurun_out/${C}_raw.csv gpurun_out/${C}_details.csv
echo done $C
