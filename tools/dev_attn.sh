#!/bin/bash
# attention parity tests + variant timings (VARIANTS="0 8" by default), two rounds
cd ${GRAFT_REPO_ROOT:-/root/repo}
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -3
for r in 1 2; do VARIANTS="${VARIANTS:-0 8}" bash tools/attn_variants.sh; done
