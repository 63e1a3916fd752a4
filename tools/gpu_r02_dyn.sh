#!/bin/bash
# Round 2: dynamic tiles + helper grid for the reserved rest-of-update.
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py -x -q -m gpu 2>&1 | tail -2
for o in ${OPTS:-"dyn_help=0" "dyn_help=1" "dyn_help=1,tail_reserve=8" "dyn_help=1,tail_reserve=24"}; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 > gpurun_out/tl_$o.txt 2>&1; head -1 gpurun_out/tl_$o.txt
done
cat "gpurun_out/tl_dyn_help=1.txt"
