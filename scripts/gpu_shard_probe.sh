export AQP_COMM_TIMEOUT_S=10 CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 200 python scripts/shard_try.py 2>&1 | tail -60
echo ==== eager
AQP_EAGER=1 timeout 200 python scripts/shard_try.py 2>&1 | tail -60
