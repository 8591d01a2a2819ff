#!/bin/bash
# evidence for one round: GPU suite, bench line, ncu launch list of the bench step, fast_kernel --set
# full at C2 x1.0, launch list of the timeline kernels at C5 x0.25
tag=${1:-r}
bash tools/gpu_final.sh $tag
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tl_launches_$tag.csv python tools/tl_time.py c5 0.25 > gpurun_out/tl_launches_$tag.log 2>&1; tail -2 gpurun_out/tl_launches_$tag.log
