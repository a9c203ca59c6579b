#!/bin/bash
# A/B of the host-buffer (e2e) path against a previous build of the C ABI: copy the package
# (+ include/) to tools/ab_old_pkg with the old sources, build it there, then run this.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OLD=$PWD/tools/ab_old_pkg/paper_2601_21444_b200/libspava_b200.so
for r in 1 2 3; do
  for arm in new old; do
    if [ $arm = old ]; then export SPAVA_LIB=$OLD; else unset SPAVA_LIB; fi
    python bench.py --no-cpu --no-extras 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$arm', round(e['value']/1e6,3), round(e['ms_per_step'],3))"
  done
done
