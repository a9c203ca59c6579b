#!/bin/bash
# ncu --set full of one C1 block-attention launch (stage 2) + stall reasons per SASS opcode
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -s 8 -c 1 \
  -o gpurun_out/attn python bench.py --steps 1 --warmup 3 --no-cpu --no-extras > gpurun_out/attn_ncu.log 2>&1
ncu -i gpurun_out/attn.ncu-rep --page source --csv --print-source sass > gpurun_out/attn_src.csv 2>/dev/null
python tools/stalls.py gpurun_out/attn_src.csv 20
ncu -i gpurun_out/attn.ncu-rep --page details --csv 2>/dev/null | grep -E "\"Duration\"|Issue Slots Busy|Executed Ipc Active|Warp Cycles Per Issued|No Eligible|Achieved Occupancy|Grid Size" | awk -F'","' '{print $13": "$15}'
