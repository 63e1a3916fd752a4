#!/bin/bash
# Sweep of the SM-reservation options of the lookahead schedule (timeline + plain timings at n=32768).
mkdir -p gpurun_out
for o in "" "pipeline_first=2" "pipeline_first=4" "pipeline_first=8" "tail_reserve=16,tail_rows=40000"; do
  f=gpurun_out/tail_$(echo "$o" | tr ',=' '__').log
  BF_OPTS="$o" timeout 300 python tools/timeline.py 32768 > $f 2>&1
  grep -E "^opts|^total" $f
done
