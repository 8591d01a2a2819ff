#!/bin/bash
# timeline: bench line (C5 x1.0 side run), launch list of the timeline kernels at C5 x0.25, full capture of tl_write
tag=${1:-r}
timeout 1200 python bench.py --no-configs --no-dropin > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; tail -c 900 gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tl_launches_$tag.csv python tools/tl_time.py c5 0.25 > gpurun_out/tl_launches_$tag.log 2>&1; tail -2 gpurun_out/tl_launches_$tag.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tl_write -c 1 -o gpurun_out/tlw_$tag python tools/tl_time.py c5 0.1 > gpurun_out/tlw_$tag.log 2>&1; tail -1 gpurun_out/tlw_$tag.log
