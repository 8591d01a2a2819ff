#!/bin/bash
# fast_kernel source-counter captures on C4 x0.25 and C5 x0.25 (where the per-record cost goes)
tag=${1:-r}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -c 1 -o gpurun_out/c4src_$tag python tools/phase_time.py c4 0.25 > gpurun_out/c4src_$tag.log 2>&1; tail -1 gpurun_out/c4src_$tag.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -c 1 -o gpurun_out/c5src_$tag python tools/phase_time.py c5 0.25 > gpurun_out/c5src_$tag.log 2>&1; tail -1 gpurun_out/c5src_$tag.log
