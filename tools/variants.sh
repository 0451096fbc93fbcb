#!/bin/bash
# Build libepfem_gpu.so variants with extra -D flags on constitutive.cu (or
# SRC="tangent.cu", or several: SRC="constitutive.cu tangent.cu") into
# paper_1805_04155_b200/lib/variants/<name>/ (tuning experiments; load one with
# EPFEM_GPU_LIB=<path>).
# usage: [SRC=tangent.cu] tools/variants.sh name "-DFOO=1" [name2 "-D..."]...
set -e
cd "$(dirname "$0")/.."
python -m paper_1805_04155_b200.build > /dev/null
P=paper_1805_04155_b200
SRC=${SRC:-constitutive.cu}
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  out=$P/lib/variants/$name; mkdir -p $out
  objs=$(ls $P/_obj/*.o)
  mine=""
  for s in $SRC; do
    FMAD=""; [ $s = constitutive.cu ] && FMAD="--fmad=false"
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -Xcompiler -ffp-contract=off --expt-relaxed-constexpr -I include $FMAD $flags \
      -c $P/csrc/$s -o $out/$s.o &
    objs=$(echo "$objs" | grep -v "/$s.o")
    mine="$mine $out/$s.o"
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libepfem_gpu.so $mine $objs -lcudart_static -ldl
  rm $mine
  echo $out/libepfem_gpu.so
done
