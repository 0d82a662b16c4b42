#!/bin/bash
# Build an A/B variant of libgpurir.so with extra -D flags into build/<name>.so (run here; the .so ships
# with the gpurun snapshot).  Load it with GPURIR_LIB=build/<name>.so.
# usage: tools/build_variant.sh <name> [-DFLAG ...]
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p build
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I include -DGPURIR_VARIANT=\"${NAME}\" "$@" -o build/${NAME}.so paper_1810_11359_b200/csrc/*.cu
