#!/bin/bash
# whole tally run per build variant (variants/lib_*.so via HAPIGPU_LIB; "" = the in-tree build)
for v in "" "$@"; do
  echo "== ${v:-default}"
  for c in "c5 0.25" "c2 1.0"; do HAPIGPU_LIB=$v timeout 200 python tools/total_time.py $c; done
done
