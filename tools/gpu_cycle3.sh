#!/bin/bash
# GPU round trip: new tests first, then the whole suite and the bench line
tag=${1:-r}
df -h /tmp > gpurun_out/box_$tag.txt
timeout 600 python -m pytest tests/test_gpu_ingest.py tests/test_gpu_distributed.py -q -x > gpurun_out/gpu_new_$tag.log 2>&1; tail -3 gpurun_out/gpu_new_$tag.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$tag.log 2>&1; tail -3 gpurun_out/gpu_tests_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
