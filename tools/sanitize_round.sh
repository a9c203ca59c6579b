#!/bin/bash
# compute-sanitizer over the GPU suites on the current code (memcheck: kernels, layer, trace,
# cpp mirror, smoke; racecheck: scorer / select / merge kernels).  Logs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py \
  tests/test_gpu_trace.py tests/test_gpu_cpp_mirror.py -q -x -m gpu -k "not peer and not nccl" \
  > gpurun_out/memcheck_gpu_suite.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_gpu_suite.log
timeout 600 $CS --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck_smoke.log
timeout 900 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_kernels.py -q -x \
  -k "score or select or merge" > gpurun_out/racecheck_score_select_merge.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/racecheck_score_select_merge.log
tail -n 4 gpurun_out/memcheck_gpu_suite.log gpurun_out/memcheck_smoke.log gpurun_out/racecheck_score_select_merge.log
