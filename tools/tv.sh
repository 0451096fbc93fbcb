#!/bin/bash
# Time library variants (tools/variants.sh) with tools/time_paths.py under gpurun:
#   tools/tv.sh "0.25 1.0" cfg4 pad0 pad4 ...
cd "$(dirname "$0")/.."
TS=$1; C=$2; shift 2
for v in "$@"; do for t in $TS; do
  echo "== $v target=$t"
  EPFEM_GPU_LIB=$PWD/paper_1805_04155_b200/lib/variants/$v/libepfem_gpu.so timeout 300 python tools/time_paths.py --target=$t $C 2>&1 | tail -1
done; done
