#!/bin/bash
# Build an A/B variant of the library with extra defines for sfk_query.cu only:
#   tools/build_qvariant.sh NAME "-DSFK_CW_NW=8 -DSFK_CW_NBK=4"
# -> paper_1701_04148_b200/_lib/NAME/libsfsketch_cuda.so (other objects from the main build)
set -e
cd "$(dirname "$0")/../paper_1701_04148_b200"
name=$1; shift
mkdir -p _build/$name _lib/$name
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $* -c csrc/sfk_query.cu -o _build/$name/sfk_query.o
objs=$(ls _build/*.o | grep -v sfk_query.o)
nvcc $ARCH -shared -o _lib/$name/libsfsketch_cuda.so $objs _build/$name/sfk_query.o -lcudart
echo built _lib/$name
