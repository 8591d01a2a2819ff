#!/bin/bash
# layout variants of fast_kernel: parity subset, then phase-1 times
for v in "$@"; do
  HAPIGPU_LIB=$v timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -x > gpurun_out/variant_$(basename $v .so).log 2>&1; echo "$v: $(tail -1 gpurun_out/variant_$(basename $v .so).log)"
done
bash tools/variant_phase.sh "$@"
