#!/bin/bash
# alternate attention variants through bench.py (isolated attention ms + step ms)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2 3; do for v in ${VARIANTS:-0 4}; do
  echo "v=$v $(SPAVA_ATTN_VARIANT=$v python bench.py --no-cpu --no-extras --steps 20 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), r["isolated"]["kernel_ms_per_step"], r["isolated"]["achieved"])')"
done; done
