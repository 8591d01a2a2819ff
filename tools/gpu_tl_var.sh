#!/bin/bash
# timeline launch lists at C5 x0.25 for the in-tree library and variants: tools/gpu_tl_var.sh tag lib...
tag=$1; shift
for v in "" "$@"; do
  n=$(basename "${v:-default}" .so)
  HAPIGPU_LIB=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tlv_${tag}_$n.csv python tools/tl_time.py c5 0.25 > /dev/null 2>&1
  echo "== $n"; python tools/ncu_summary.py launches gpurun_out/tlv_${tag}_$n.csv | sed -n 2,7p
done
