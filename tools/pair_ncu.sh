#!/bin/bash
# ncu --set full of one attention launch per kernel form (1-CTA, pair with P in TMEM, pair with
# P in smem; dev build) on tools/attn_bench.py -> gpurun_out/pair{0,1,2}.ncu-rep
cd ${GRAFT_REPO_ROOT:-/root/repo}
for pr in 0 1 2; do
SPAVA_ATTN_PAIR=$pr timeout 300 ncu --set full --import-source on --clock-control none -k regex:"attn_" -s 4 -c 1 -o gpurun_out/pair$pr python tools/attn_bench.py > /dev/null 2>&1
done
ls gpurun_out/pair*
