cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python tools/score_ab.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/score_l.csv python tools/score_ab.py > /dev/null 2>&1
python tools/ktimes.py gpurun_out/score_l.csv
ncu --set full --import-source on --clock-control none -k regex:logits_kernel -c 2 -o gpurun_out/logits_full python tools/score_ab.py > /dev/null 2>&1
ls -la gpurun_out
