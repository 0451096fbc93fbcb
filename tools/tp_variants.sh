#!/bin/bash
# tools/time_paths.py over variant libraries: CFGS="cfg4 cfg3" bash tools/tp_variants.sh name1 name2 ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ $v = default ]; then L="EPFEM_X=1"; else L="EPFEM_GPU_LIB=paper_1805_04155_b200/lib/variants/$v/libepfem_gpu.so"; fi
  for c in ${CFGS:-cfg4}; do
    echo "== $v $c" >> gpurun_out/tp_summary.txt
    env $L timeout 900 python tools/time_paths.py ${TARGET:+--target=$TARGET} $c 2>> gpurun_out/tp_err.txt | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()})" >> gpurun_out/tp_summary.txt
  done
done
