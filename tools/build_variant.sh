#!/bin/bash
# Build an A/B variant of the library with extra defines for ONE source file:
#   tools/build_variant.sh NAME SRC "-DFOO=1 -DBAR=2"     (SRC e.g. sfk_sf.cu)
# -> paper_1701_04148_b200/_lib/NAME/libsfsketch_cuda.so (other objects from the main build)
set -e
cd "$(dirname "$0")/../paper_1701_04148_b200"
name=$1; src=$2; shift 2
obj=${src%.cu}.o
mkdir -p _build/$name _lib/$name
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $* -c csrc/$src -o _build/$name/$obj
objs=$(ls _build/*.o | grep -v "/$obj")
nvcc $ARCH -shared -o _lib/$name/libsfsketch_cuda.so $objs _build/$name/$obj -lcudart
echo built _lib/$name
