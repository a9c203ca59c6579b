#!/bin/bash
# A/B an environment knob on the e2e (host-buffer) step: ENVVAR=NAME VALUES="1 2" bash tools/ab_e2e_env.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2 3; do for v in ${VALUES:-0 1}; do
  env $ENVVAR=$v timeout 300 python bench.py --no-cpu --no-extras --no-sweep 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$ENVVAR=$v', 'e2e', round(e['value']/1e6,3), round(e['ms_per_step'],3), 'floor', e.get('copy_floor_ms'), 'same', e.get('outputs_equal_device_path'), 'dev', round(d['ms_per_step'],3))"
done; done
