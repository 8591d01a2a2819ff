#!/bin/bash
# one GPU round trip while iterating on the range kernel: parity tests, phase-1 timing, one ncu capture
tag=${1:-x}
timeout 400 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/fast_tests_$tag.log 2>&1; tail -4 gpurun_out/fast_tests_$tag.log
timeout 200 python tools/phase_time.py c2 1.0 > gpurun_out/pt_$tag.log 2>&1; tail -2 gpurun_out/pt_$tag.log
if [ "$2" != "noprof" ]; then
timeout 300 ncu --set full --import-source on --clock-control none -k regex:fast_kernel -c 1 -o gpurun_out/fast_$tag python tools/phase_time.py c2 0.25 > gpurun_out/ncu_$tag.log 2>&1; tail -1 gpurun_out/ncu_$tag.log
fi
