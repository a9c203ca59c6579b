#!/bin/bash
# attention A/B on the GPU box: variant parity tests, then alternating kernel timings
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -2
for rep in 1 2; do for v in ${VARIANTS:-0 2 3 6}; do
  SPAVA_ATTN_VARIANT=$v timeout 300 python tools/attn_bench.py 2>&1 | tail -1
done; done
SPAVA_ATTN_VARIANT=1 timeout 300 python tools/attn_bench.py 2>&1 | tail -3
