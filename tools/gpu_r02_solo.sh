#!/bin/bash
# one-warp-per-32-rows persistent fused TRSM subtree (trsm_warp=2) vs the 4-warp groups (1)
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_trsm or trsm" 2>&1 | tail -2
for o in trsm_warp=1 trsm_warp=2; do
  BF_OPTS=$o python tools/prof_diag.py 2048 5 | sed "s/^/$o /"
done
for r in 1 2; do for o in trsm_warp=1 trsm_warp=2; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 | grep -E "opts|total"
done; done
for o in trsm_warp=1 trsm_warp=2; do BF_OPTS=$o python tools/c4_tree_sweep.py 32768 1024 2>&1 | head -1 | sed "s/^/$o /"; done
