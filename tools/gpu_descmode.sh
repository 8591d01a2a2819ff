#!/bin/bash
# C4 (4k-schema registry): inline descriptors in shared memory (8 B) vs through L1; correctness of the single pass
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -x > gpurun_out/descmode_tests.log 2>&1; tail -2 gpurun_out/descmode_tests.log
for m in 2 0; do echo "== desc mode <= $m"; for c in "c4 0.25" "c2 1.0"; do HAPIGPU_DESC_MODE=$m timeout 300 python tools/phase_time.py $c | tail -1; done; done
