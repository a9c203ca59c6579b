#!/bin/bash
# Round profile on the GPU box: launch list of a bench run + one `ncu --set full` capture of
# a whole bench step (9 launches: the 4th of 4 steps).  Summarise here with
#   python tools/ncu_summary.py gpurun_out/step_full.ncu-rep profiles/r02_ncu_step C1
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-extras --no-sweep > gpurun_out/b_ncu.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"attn_fwd|logits|rowstats|colsum|select|gather|merge" --launch-skip 27 -c 9 \
  -o gpurun_out/step_full python bench.py --steps 1 --warmup 3 --no-cpu --no-extras --no-sweep > gpurun_out/step_full.log 2>&1
tail -2 gpurun_out/step_full.log
