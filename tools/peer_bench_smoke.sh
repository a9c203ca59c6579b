#!/bin/bash
# N=2 bench path with the peer fabric, both ranks on cuda:0 (smoke of the N>1 code path;
# the timing is meaningless -- two ranks share one GPU)
set -o pipefail
mkdir -p gpurun_out
SPAVA_BENCH_ONE_GPU=1 CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python -m torch.distributed.run \
  --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-extras > gpurun_out/peer_bench_n2.log 2>&1
echo "rc=$?" >> gpurun_out/peer_bench_n2.log
tail -c 3000 gpurun_out/peer_bench_n2.log
