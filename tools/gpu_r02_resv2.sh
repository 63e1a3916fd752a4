#!/bin/bash
cd "$(dirname "$0")/.."
for o in ${OPTS:-"" "reserve_extra=2" "reserve_extra=6" "reserve_extra=8" "reserve_min=8" "reserve_extra=6,reserve_min=16"}; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 | grep -E "opts|total" | paste - -
done
