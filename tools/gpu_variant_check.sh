#!/bin/bash
# a fast.cu build variant: the single-pass parity tests under it, then phase-1 timing against the in-tree build
v=$1; tag=$2
HAPIGPU_LIB=$v timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_golden.py -q -x > gpurun_out/variant_$tag.log 2>&1; tail -3 gpurun_out/variant_$tag.log
bash tools/variant_phase.sh $v
