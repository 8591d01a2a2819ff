#!/bin/bash
# phase-1 times on C2 / C4 / C5 at full size, then the GPU suite
tag=${1:-r}
for c in c2 c4 c5; do timeout 300 python tools/phase_time.py $c 1.0 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$tag.log 2>&1; tail -3 gpurun_out/gpu_tests_$tag.log
