#!/bin/bash
# phase-1 times of build variants on C2 / C5 x1.0 ("" = in-tree)
for v in "" "$@"; do echo "== ${v:-default}"; for c in "c2 1.0" "c5 1.0"; do HAPIGPU_LIB=$v timeout 300 python tools/phase_time.py $c 2>&1 | tail -1; done; done
