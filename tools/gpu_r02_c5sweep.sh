#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for o in "group=8" "group=4" "group=16" "group=32" "tiles_per_cta=2" "tiles_per_cta=4" "persist=1" "tma_variant=3" "tma_variant=0"; do
  BF_OPTS=$o timeout 300 python tools/c5_tmem.py 128 2 1 2>&1 | tail -1
done
