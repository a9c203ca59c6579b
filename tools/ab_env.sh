#!/bin/bash
# A/B an environment knob on the device-path bench step: ENVVAR=NAME VALUES="0 1" bash tools/ab_env.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2 3; do for v in ${VALUES:-0 1}; do
  env $ENVVAR=$v timeout 300 python bench.py --no-cpu --no-extras --no-sweep 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$ENVVAR=$v', round(d['value']/1e6,3), round(d['ms_per_step'],4), 'attn', r['kernel_ms_per_step'], 'score', r['score_ms_per_step'], 'iso', r['isolated']['kernel_ms_per_step'], r['isolated']['score_ms_per_step'], 'e2e', round(d['e2e']['ms_per_step'],3))"
done; done
