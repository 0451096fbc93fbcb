#!/bin/bash
# time lib/variants/<name> builds on one config: CFG=cfg5 bash tools/sweep_variants.sh name1 name2 ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C=${CFG:-cfg5}
for v in default "$@"; do
  # name, EPFEM_A=x,EPFEM_B=y (env only) or name+EPFEM_A=x (variant library plus env)
  if [ $v = default ]; then L="EPFEM_X=1"; elif [[ $v == EPFEM_* ]]; then L=$(echo $v | tr ',' ' ');
  else L="EPFEM_GPU_LIB=paper_1805_04155_b200/lib/variants/${v%%+*}/libepfem_gpu.so"
    [[ $v == *+* ]] && L="$L $(echo ${v#*+} | tr ',' ' ')"; fi
  env $L EPFEM_X=1 timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/sweep_$v.json 2> gpurun_out/sweep_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/sweep_$v.json').read().strip().splitlines()[-1]); print('$C $v', round(d['ms_per_step'],3), {k[:14]: round(x,3) for k,x in d['kernels_ms'].items()})" >> gpurun_out/sweep_summary.txt 2>&1
done
