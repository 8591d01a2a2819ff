#!/bin/bash
# GPU round trip: parity suite, bench line (N=1), the N=2 bench path on one GPU over gloo, box facts
tag=${1:-r}
nproc > gpurun_out/box_$tag.txt; free -g >> gpurun_out/box_$tag.txt; nvidia-smi -L >> gpurun_out/box_$tag.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_$tag.log 2>&1; tail -3 gpurun_out/gpu_tests_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --backend gloo --scale 0.02 --steps 3 --warmup 3 > gpurun_out/bench2_$tag.json 2> gpurun_out/bench2_$tag.err; echo "bench2 rc=$?"; tail -c 600 gpurun_out/bench2_$tag.json; tail -5 gpurun_out/bench2_$tag.err
