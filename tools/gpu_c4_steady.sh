#!/bin/bash
# C4 x1.0 steady-state fast_kernel (the deep-stack variant the host picks after the first run)
tag=${1:-r}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 3 -c 1 -o gpurun_out/c4st_$tag python tools/phase_time.py c4 1.0 > gpurun_out/c4st_$tag.log 2>&1; tail -1 gpurun_out/c4st_$tag.log
