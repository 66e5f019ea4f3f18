#!/bin/bash
# Exercise bench.py's N>1 (row-sharded C5) code path on a ONE-GPU box: two
# ranks share cuda:0 over gloo + CUDA IPC on a small C5-shaped instance.
export AQP_BENCH_TEST_N=200000 AQP_BENCH_TEST_BACKEND=gloo AQP_COMM_TIMEOUT_S=60 AQP_BENCH_NO_SECONDARY=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline 2>&1 | grep -v Warning | tail -5
