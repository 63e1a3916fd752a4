#!/bin/bash
# C2: the first panel as the fused factor with per-column release (fused_first = % of SMs)
cd "$(dirname "$0")/.."
for r in 1 2; do
  for o in fused_first=0 fused_first=100 fused_first=66 fused_first=50; do
    BF_OPTS=$o timeout 300 python tools/timeline.py 32768 > /tmp/tl.txt 2>&1
    echo "$(grep opts /tmp/tl.txt) | step0 col_done $(awk '$1=="0"{print $3}' /tmp/tl.txt) | $(grep total /tmp/tl.txt)"
  done
done
