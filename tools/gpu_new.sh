#!/bin/bash
# GPU round trip: the named test files first (-x), then the whole GPU suite
tag=$1; shift
timeout 900 python -m pytest "$@" -q -x > gpurun_out/gpu_new_$tag.log 2>&1; tail -3 gpurun_out/gpu_new_$tag.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$tag.log 2>&1; tail -3 gpurun_out/gpu_tests_$tag.log
