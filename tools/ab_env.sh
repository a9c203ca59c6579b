#!/bin/bash
# A/B an environment switch through bench.py on one box, alternating: ENVS="A=0 A=1" bash tools/ab_env.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2 3; do for e in ${ENVS}; do
  echo "$e $(env $e python bench.py --no-cpu --no-extras --steps 20 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), r["kernel_ms_per_step"], r["isolated"]["kernel_ms_per_step"], r["isolated"]["merge_ms_per_step"])')"
done; done
