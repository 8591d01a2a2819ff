#!/bin/bash
# timeline change: timeline parity tests, then timings at C5 x0.25 (tl_time) and a launch list
tag=${1:-r}
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_distributed.py -m gpu -q -x -k "timeline or golden or tl" > gpurun_out/tlchk_$tag.log 2>&1; tail -3 gpurun_out/tlchk_$tag.log
timeout 300 python tools/tl_time.py c5 0.25 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tl_launches_$tag.csv python tools/tl_time.py c5 0.25 > gpurun_out/tl_launches_$tag.log 2>&1; tail -1 gpurun_out/tl_launches_$tag.log
