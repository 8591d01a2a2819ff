#!/bin/bash
# build variants/lib_<name>.so: fast.cu with extra -D flags, the other objects from the in-tree build
# usage: tools/build_variant.sh name "-DFLAG1 -DFLAG2"
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants
B=paper_2504_03683_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I include $@ -c -o variants/fast_$name.o paper_2504_03683_b200/csrc/fast.cu
objs=$(ls $B/*.o | grep -v "/fast.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$name.so variants/fast_$name.o $objs
echo variants/lib_$name.so
