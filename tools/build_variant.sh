#!/bin/bash
# Build a variant of the library from a modified copy of csrc (A/B experiments).
#   tools/build_variant.sh NAME   (after copying/editing _variants/NAME/pkg/csrc/*)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
V=$ROOT/_variants/$1
mkdir -p $V/include
cp $ROOT/include/*.h $V/include/
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -diag-suppress 177 -o $V/lib.so $V/pkg/csrc/ehmg_solver.cu -lcusolver -lcublas \
  -Xlinker -rpath,/usr/local/cuda/lib64
echo $V/lib.so
