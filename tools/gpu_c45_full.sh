#!/bin/bash
# C4 / C5 at full size: phase-1 times, then fast_kernel source-counter captures (where the per-record cost goes)
tag=${1:-r}
for c in c4 c5; do timeout 300 python tools/phase_time.py $c 1.0 2>&1 | tail -1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 1 -c 1 -o gpurun_out/c4src_$tag python tools/phase_time.py c4 1.0 > gpurun_out/c4src_$tag.log 2>&1; tail -1 gpurun_out/c4src_$tag.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 1 -c 1 -o gpurun_out/c5src_$tag python tools/phase_time.py c5 1.0 > gpurun_out/c5src_$tag.log 2>&1; tail -1 gpurun_out/c5src_$tag.log
