#!/bin/bash
# ncu --set full of the exact scorer's kernels (one C1 block each) + per-kernel pipe summary
# and stall reasons per SASS opcode for each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"logits|combine|colsum" -s 3 -c 3 \
  -o gpurun_out/score_full python tools/score_bench.py > gpurun_out/score_ncu.log 2>&1
ncu -i gpurun_out/score_full.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/score_raw.csv
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/score_raw.csv')))
h=rows[0]
keys=["Kernel Name","gpu__time_duration.sum","sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active","sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
"smsp__issue_active.avg.pct_of_peak_sustained_active","sm__warps_active.avg.pct_of_peak_sustained_active",
"launch__registers_per_thread","gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed","launch__occupancy_limit_registers",
"smsp__average_warp_latency_issue_stalled_short_scoreboard","sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    print(" | ".join(f"{k.split('.')[0][-28:]}={r[h.index(k)]}" for k in keys if k in h))
PY
for i in 1 2 3; do
  ncu -i gpurun_out/score_full.ncu-rep --page source --csv --print-source sass --launch-skip $((i-1)) --launch-count 1 > gpurun_out/score_src$i.csv 2>/dev/null
  echo "== kernel $i"; python tools/stalls.py gpurun_out/score_src$i.csv 10
done
