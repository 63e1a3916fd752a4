#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "half_width or variants or red_fold or persist or reserv" 2>&1 | tail -2
for o in tma_wt=32 tma_wt=64; do
  echo "$o: $(python tools/prof_chol.py syrk 30720 2048 $o 2>/dev/null | tail -1)"
  echo "$o: $(python tools/prof_chol.py syrk 16384 2048 $o 2>/dev/null | tail -1)"
done
for r in 1 2; do for o in tma_wt=32 tma_wt=64 tma_bn=128; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 | grep opts
done; done
