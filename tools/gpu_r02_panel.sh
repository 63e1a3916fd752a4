#!/bin/bash
# C2 with the panel tile order of the trailing GEMMT (BF_OPTS=panel_tiles=w)
cd "$(dirname "$0")/.."
for o in ${OPTS:-"panel_tiles=0" "panel_tiles=8" "panel_tiles=16" "panel_tiles=32"}; do
  BF_OPTS=$o timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$o', d['ms_per_step'], d['step_ms'])"
done
