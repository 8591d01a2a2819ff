#!/bin/bash
# build variants/lib_<name>.so from ALL translation units with extra -D flags (layout-changing variants)
# usage: tools/build_variant_all.sh name "-DFLAG1 -DFLAG2"
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants/obj_$name
objs=""
for src in paper_2504_03683_b200/csrc/*.cu; do
  o=variants/obj_$name/$(basename $src .cu).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I include $@ -c -o $o $src &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$name.so $objs
echo variants/lib_$name.so
