#!/bin/bash
# overlapped panel (diag factor || TRSM of the rows below): tests, diag/timeline A/B
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "overlap or reservation or lookahead or fused_trsm" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_headline_parity.py -x -q -m gpu 2>&1 | tail -2
for r in 1 2; do for o in ${OPTS:-panel_overlap=0 panel_overlap=1}; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 > gpurun_out/tl_$o.txt; grep -E "opts|total" gpurun_out/tl_$o.txt
done; done
cat gpurun_out/tl_panel_overlap=1.txt | head -20
