#!/bin/bash
# quick GPU loop for scorer work: scorer/select parity, scorer timing, full-size parity,
# a short bench line and its launch list
cd ${GRAFT_REPO_ROOT:-/root/repo}; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "score or select or needle" > gpurun_out/t_score.log 2>&1; tail -3 gpurun_out/t_score.log
timeout 300 python tools/score_bench.py 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity_full.py -q -x > gpurun_out/t_full.log 2>&1; tail -3 gpurun_out/t_full.log
timeout 300 python bench.py --no-cpu --no-extras --no-sweep > gpurun_out/bench_s.json 2>gpurun_out/bench_s.err; python -c "
import json;d=json.load(open('gpurun_out/bench_s.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['score_ms_per_step'],r['isolated'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras --no-sweep > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_s.csv | tail -9
