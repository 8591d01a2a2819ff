#!/bin/bash
# timeline device time per build variant (variants/lib_*.so via HAPIGPU_LIB; "" = the in-tree build)
for v in "" "$@"; do
  echo "== ${v:-default}"; HAPIGPU_LIB=$v timeout 200 python tools/tl_time.py c5 0.1 2>&1 | grep -oE "tile kernel [0-9.]+ ms|timeline [0-9.]+ ms"
done
