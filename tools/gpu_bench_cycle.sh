#!/bin/bash
# full GPU round trip: parity suite, bench line, ncu launch list and DRAM traffic of the phase-1 kernels
tag=${1:-r}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$tag.log 2>&1; tail -3 gpurun_out/gpu_tests_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 600 gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 1 --no-timeline --no-configs > gpurun_out/bench_ncu_$tag.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fast_ --csv --log-file gpurun_out/traffic_$tag.csv python tools/phase_time.py c2 1.0 > gpurun_out/traffic_$tag.log 2>&1
ls -la gpurun_out | tail -5
