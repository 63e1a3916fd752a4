#!/bin/bash
# C2 timeline: launch sequence vs fused (=2) with the fused grid at a share of the reserved SMs
cd "$(dirname "$0")/.."
for r in 1 2; do
  for o in fused_diag=1 fused_diag=2,fused_diag_pct=50 fused_diag=2,fused_diag_pct=33 fused_diag=2,fused_diag_pct=66; do
    BF_OPTS=$o timeout 300 python tools/timeline.py 32768 | grep -E "opts|total" | tr '\n' ' '; echo
  done
done
