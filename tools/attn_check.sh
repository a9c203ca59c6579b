#!/bin/bash
# attention dev loop on the GPU box: parity tests + kernel timing per variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for v in ${VARIANTS:-0 1}; do
  echo "== variant $v: $(SPAVA_ATTN_VARIANT=$v timeout 600 python -m pytest tests -m gpu -x -q -k "${TESTK:-attention or layer or dense}" 2>&1 | tail -1)"
  SPAVA_ATTN_VARIANT=$v timeout 300 python tools/attn_bench.py 2>&1 | tail -2
done
