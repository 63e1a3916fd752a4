#!/bin/bash
# fused diagonal factor inside the overlapped panels (fused_diag=2, stream-memory-wait release) vs the
# launch sequence (1): parity, C2 timeline, C4
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_diag" 2>&1 | tail -3
for r in 1 2; do
  for o in fused_diag=1 fused_diag=2; do
    BF_OPTS=$o timeout 300 python tools/timeline.py 32768 | grep -E "opts|total" | sed "s/^/$o /"
  done
done
BF_OPTS=fused_diag=2 timeout 300 python tools/timeline.py 32768 | tail -18
for o in fused_diag=1 fused_diag=2 fused_diag=1 fused_diag=2; do BF_OPTS=$o timeout 300 python tools/bench_mixed.py 32768 2048 2>/dev/null | head -1 | cut -c1-260; done
