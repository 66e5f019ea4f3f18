#!/bin/bash
# Exercise bench.py's N>1 (row-sharded) code path on a ONE-GPU box: two ranks
# share cuda:0 over gloo + CUDA IPC, a small C2-shaped instance, few windows.
export AQP_BENCH_TEST_N=20000 AQP_BENCH_TEST_ITERS=640 AQP_BENCH_TEST_BACKEND=gloo AQP_COMM_TIMEOUT_S=60
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -v Warning | tail -5
