#!/bin/bash
# SM reservation default (tail_reserve=16 when the rest of the update is <= 32768 rows) vs variants at n=131072.
mkdir -p gpurun_out
for o in "" "tail_rows=65536" "tail_rows=1000000,reserve_strided=1"; do
  BF_OPTS="$o" timeout 600 python tools/bench_c3_single.py 131072 4096 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$o]', d['ms'], d['tflops'], d['rel_residual_Ax_vs_LLtx'])"
done
BF_OPTS="" timeout 300 python tools/timeline.py 32768 2>&1 | grep -E "^opts"
