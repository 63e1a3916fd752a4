#!/bin/bash
# early panels (diagonal factor of panel k+1 under the rest of the column update) A/B, C2 timeline
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do for o in ${OPTS:-early_panel=0 early_panel=1 early_panel=2 early_panel=3}; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 > gpurun_out/tl.txt; grep -E "opts|total" gpurun_out/tl.txt | paste - -
done; done
