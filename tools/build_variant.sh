#!/bin/bash
# Build a variant of the library with extra nvcc defines into paper_2408_01331_b200/_lib/variants/NAME
# usage: bash tools/build_variant.sh NAME SOURCE.cu -DFOO [-DBAR ...]   (debug tool)
set -e
cd "$(dirname "$0")/../paper_2408_01331_b200/_lib"
name=$1; src=$2; shift 2
rm -rf variants/$name && mkdir -p variants/$name && cp *.o variants/$name/
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -I ../../include \
  -c ../csrc/$src -o variants/$name/${src%.cu}.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libhnn_b200.so variants/$name/*.o -lcuda
echo variants/$name/libhnn_b200.so
