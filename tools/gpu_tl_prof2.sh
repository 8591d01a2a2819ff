#!/bin/bash
# full captures with source of the timeline formatting kernels at C5 x0.25
tag=${1:-r}
for k in ${2:-tl_write tl_len}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/${k}_$tag python tools/tl_time.py c5 0.25 > gpurun_out/${k}_$tag.log 2>&1; tail -1 gpurun_out/${k}_$tag.log
done
