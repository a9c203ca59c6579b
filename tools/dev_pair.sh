#!/bin/bash
# CTA-pair attention (SPAVA_ATTN_PAIR=1): parity tests + timings against the 1-CTA kernel
cd ${GRAFT_REPO_ROOT:-/root/repo}
SPAVA_ATTN_PAIR=${TESTPAIR:-1} timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_matches or single_key or deterministic" 2>&1 | tail -4
for r in 1 2; do
  for pr in ${PAIRS:-0 1}; do echo -n "pair=$pr "; SPAVA_ATTN_PAIR=$pr timeout 120 python tools/attn_bench.py 2>&1 | grep variant; done
done
