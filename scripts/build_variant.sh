#!/bin/bash
# Build a compile-time variant of the engine library for A/B timing:
#   scripts/build_variant.sh NAME -DFLAG=VALUE ...   ->  paper_2402_03060_b200/_build/variants/NAME.so
# then run with UH_LIB_PATH=paper_2402_03060_b200/_build/variants/NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p paper_2402_03060_b200/_build/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -ccbin /usr/bin/g++ "$@" \
  -o paper_2402_03060_b200/_build/variants/$name.so paper_2402_03060_b200/csrc/*.cu -lcufft
echo paper_2402_03060_b200/_build/variants/$name.so
