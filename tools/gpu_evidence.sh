#!/bin/bash
# evidence run: GPU suite, bench line, timeline launch list at C5 x0.25, tl_write --set full
tag=${1:-r}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$tag.log 2>&1; tail -2 gpurun_out/gpu_tests_$tag.log
timeout 1200 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tl_launches_$tag.csv python tools/tl_time.py c5 0.25 > gpurun_out/tl_launches_$tag.log 2>&1; tail -1 gpurun_out/tl_launches_$tag.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tl_write -c 1 -o gpurun_out/tl_write_$tag python tools/tl_time.py c5 0.25 > gpurun_out/tl_write_$tag.log 2>&1; tail -1 gpurun_out/tl_write_$tag.log
