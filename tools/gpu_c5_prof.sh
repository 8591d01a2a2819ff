#!/bin/bash
# C5 x1.0 steady-state fast_kernel source counters (the device-record drain)
tag=${1:-r}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 2 -c 1 -o gpurun_out/c5st_$tag python tools/phase_time.py c5 1.0 > gpurun_out/c5st_$tag.log 2>&1; tail -1 gpurun_out/c5st_$tag.log
