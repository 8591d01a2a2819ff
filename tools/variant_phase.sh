#!/bin/bash
# phase-1 (fast_kernel) time per build variant on C2 x1 and C5 x0.25 ("" = the in-tree build)
for v in "" "$@"; do
  echo "== ${v:-default}"
  for c in "c2 1.0" "c5 0.25"; do HAPIGPU_LIB=$v timeout 300 python tools/phase_time.py $c 2>&1 | tail -1; done
done
