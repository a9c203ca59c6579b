#!/bin/bash
# every attention variant through tools/attn_bench.py (C1 block-hi shape, dense causal 32K, full 16K);
# variants other than 0 need a dev build: SPAVA_DEV_VARIANTS=1 python -m paper_2601_21444_b200.build --force
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in ${VARIANTS:-0 1 2 3 4 5 6 7 8 9 10 11 12 13 14}; do
  SPAVA_ATTN_VARIANT=$v timeout 120 python tools/attn_bench.py 2>&1 | grep -v Warning | tail -4
done
