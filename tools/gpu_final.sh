#!/bin/bash
# round-end evidence: GPU suite, bench line, ncu launch list of the bench step, fast_kernel --set full at C2 x1.0
tag=${1:-r}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$tag.log 2>&1; tail -2 gpurun_out/gpu_tests_$tag.log
timeout 1200 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; tail -c 200 gpurun_out/bench_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 --no-timeline --no-configs --no-dropin > gpurun_out/launches_$tag.log 2>&1; tail -1 gpurun_out/launches_$tag.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 2 -c 1 -o gpurun_out/fastfull_$tag python tools/phase_time.py c2 1.0 > gpurun_out/fastfull_$tag.log 2>&1; tail -1 gpurun_out/fastfull_$tag.log
