#!/bin/bash
# timeline kernels at C5 x0.25: launch list + full captures with source of the top kernels
tag=${1:-r}
sc=${2:-0.25}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tl_launches_$tag.csv python tools/tl_time.py c5 $sc > gpurun_out/tl_launches_$tag.log 2>&1; tail -2 gpurun_out/tl_launches_$tag.log
for k in tl_write tl_len seg_decode tl_merge; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/${k}_$tag python tools/tl_time.py c5 $sc > gpurun_out/${k}_$tag.log 2>&1; tail -1 gpurun_out/${k}_$tag.log
done
