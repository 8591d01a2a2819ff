#!/bin/bash
# fast_kernel: --set full with source counters at C2 x0.25 (per-SASS-line executed instructions / stalls)
tag=${1:-r}
timeout 300 python -m pytest tests/test_gpu_ingest.py -q -x > gpurun_out/gpu_ingest_$tag.log 2>&1; tail -2 gpurun_out/gpu_ingest_$tag.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -c 1 -o gpurun_out/fastsrc_$tag python tools/phase_time.py c2 0.25 > gpurun_out/fastsrc_$tag.log 2>&1; tail -2 gpurun_out/fastsrc_$tag.log
