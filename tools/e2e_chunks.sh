#!/bin/bash
# A/B of host-buffer row-chunk tables (SPAVA_COPY_CHUNKS, fractions of 32 of a block) on e2e
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TABLES=${TABLES:-"0,2,8,16,24,32 0,2,4,8,12,16,20,26,32 0,1,2,4,6,8,12,16,20,24,28,32 0,1,3,6,10,14,18,22,27,32"}
for r in 1 2; do for t in $TABLES; do
  SPAVA_COPY_CHUNKS=$t timeout 300 python bench.py --no-cpu --no-extras --no-sweep 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$t', round(e['value']/1e6,3), round(e['ms_per_step'],3), 'floor', e.get('copy_floor_ms'), 'dev', round(d['ms_per_step'],3))"
done; done
