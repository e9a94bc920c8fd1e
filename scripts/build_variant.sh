#!/bin/bash
# Build a compile-time variant of the engine library for A/B timing:
#   scripts/build_variant.sh NAME SRC.cu -DFLAG=VALUE ...  ->  paper_2402_03060_b200/_build/variants/NAME.so
# SRC.cu (a file under csrc/) is recompiled with the flags; every other object comes from the
# regular build (python -m paper_2402_03060_b200.build).  Run with UH_LIB_PATH=<the .so>.
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
B=paper_2402_03060_b200/_build
mkdir -p $B/variants
base=$(basename "$src" .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -ccbin /usr/bin/g++ "$@" \
  -c -o $B/variants/$name.$base.o paper_2402_03060_b200/csrc/$base.cu
objs=$(ls $B/*.o | grep -v "/$base.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ \
  -o $B/variants/$name.so $objs $B/variants/$name.$base.o
echo $B/variants/$name.so
