#!/bin/bash
# timeline from the single pass: parity tests, then tally and timeline timings (exact path baseline via HAPIGPU_TL_EXACT)
tag=${1:-r}
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -x -k "timeline or golden or tl" > gpurun_out/tlfast_$tag.log 2>&1; tail -3 gpurun_out/tlfast_$tag.log
timeout 300 python tools/phase_time.py c2 1.0 2>&1 | tail -1
timeout 300 python tools/phase_time.py c5 0.25 2>&1 | tail -1
echo "== single pass"; HAPIGPU_DEBUG=1 timeout 300 python tools/tl_time.py c5 0.25 2>&1 | tail -3
echo "== exact"; HAPIGPU_TL_EXACT=1 timeout 300 python tools/tl_time.py c5 0.25 2>&1 | tail -2
