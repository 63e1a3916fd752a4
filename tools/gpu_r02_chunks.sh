#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_graph.py -x -q -m gpu -k "overlap or graph or lookahead" 2>&1 | tail -2
for r in 1 2; do for o in ${OPTS:-"panel_chunks=1" "panel_chunks=2" "panel_chunks=4" "panel_chunks=4,panel_chunk_rows=2048"}; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 > gpurun_out/tlc.txt; echo "$o $(grep -E 'opts|total' gpurun_out/tlc.txt | paste - - | cut -c1-150)"; grep -E "^   0 " gpurun_out/tlc.txt
done; done
