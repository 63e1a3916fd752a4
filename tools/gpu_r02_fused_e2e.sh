#!/bin/bash
# fused diagonal factor on/off: C2 timeline (plain + per-step) and C4 factor
cd "$(dirname "$0")/.."
for r in 1 2; do
  for o in fused_diag=0 fused_diag=1; do
    BF_OPTS=$o timeout 300 python tools/timeline.py 32768 | grep -E "opts|total" | sed "s/^/$o /"
  done
done
BF_OPTS=fused_diag=1 timeout 300 python tools/timeline.py 32768 | tail -18
for o in fused_diag=0 fused_diag=1 fused_diag=0 fused_diag=1; do BF_OPTS=$o timeout 300 python tools/bench_mixed.py 32768 2048 | head -1 | cut -c1-300; done
