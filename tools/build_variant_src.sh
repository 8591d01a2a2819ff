#!/bin/bash
# build variants/lib_<name>.so: one source (csrc/<src>.cu) with extra -D flags, the other objects from the in-tree build
# usage: tools/build_variant_src.sh name src "-DFLAG1 -DFLAG2"
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
mkdir -p variants
B=paper_2504_03683_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I include $@ -c -o variants/${src}_$name.o paper_2504_03683_b200/csrc/$src.cu
objs=$(ls $B/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$name.so variants/${src}_$name.o $objs
echo variants/lib_$name.so
