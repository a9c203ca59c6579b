#!/bin/bash
# ncu --set full of one logits_kernel launch (C1 block) + stall reasons per SASS opcode
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:logits_kernel -s 2 -c 1 \
  -o gpurun_out/logits python tools/score_bench.py > gpurun_out/logits_ncu.log 2>&1
ncu -i gpurun_out/logits.ncu-rep --page source --csv --print-source sass > gpurun_out/logits_src.csv 2>/dev/null
python tools/stalls.py gpurun_out/logits_src.csv 14
ncu -i gpurun_out/logits.ncu-rep --page details --csv 2>/dev/null | grep -E "Issue Slots Busy|Executed Ipc Active|Warp Cycles Per Issued|No Eligible|Achieved Occupancy|Duration|Registers Per|Local Memory|Bank Conflicts|Shared Load|Fused" | cut -c1-220
