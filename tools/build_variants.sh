#!/bin/bash
# Build library variants that differ in -D flags (A/B experiments):
#   tools/build_variants.sh name1:"-DX=1 -DY=2" name2:"..."   -> _variants/lib_<name>.so
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p $ROOT/_variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
      -diag-suppress 177 $flags -o $ROOT/_variants/lib_$name.so $ROOT/paper_2307_03242_b200/csrc/ehmg_solver.cu \
      -lcusolver -lcublas -Xlinker -rpath,/usr/local/cuda/lib64 && echo built $name ) &
done
wait
