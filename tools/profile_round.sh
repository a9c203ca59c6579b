#!/bin/bash
# Round profile on the GPU box: launch list of a bench run + one `ncu --set full` capture of
# a whole bench step (12 launches after 3 warm-up steps).  Summarise here with
#   python tools/ncu_summary.py gpurun_out/step_full.ncu-rep profiles/r01_ncu_step C1
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > gpurun_out/b_ncu.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"attn_fwd|logits|rowstats|colsum|select|gather|merge" --launch-skip 36 -c 12 \
  -o gpurun_out/step_full python bench.py --steps 1 --warmup 3 --no-cpu --no-extras > gpurun_out/step_full.log 2>&1
tail -2 gpurun_out/step_full.log
