#!/bin/bash
# scorer dev loop on the GPU box: parity tests + per-kernel launch times
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "score or select or layer or golden" 2>&1 | tail -4 > gpurun_out/sc_pytest.log; cat gpurun_out/sc_pytest.log
timeout 300 python tools/score_bench.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/score_l.csv python tools/score_bench.py > /dev/null 2>&1
python tools/ktimes.py gpurun_out/score_l.csv
