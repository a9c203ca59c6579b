#!/bin/bash
# N>1 bench path with the peer fabric, all ranks on cuda:0 (smoke of the N>1 code path;
# the timing is meaningless -- the ranks share one GPU).  N defaults to 2 (C1); N=4 runs C2.
set -o pipefail
N=${N:-2}
mkdir -p gpurun_out
SPAVA_BENCH_ONE_GPU=1 CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python -m torch.distributed.run \
  --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 3 --warmup 3 --no-cpu > gpurun_out/peer_bench_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/peer_bench_n$N.log
tail -c 1500 gpurun_out/peer_bench_n$N.log
