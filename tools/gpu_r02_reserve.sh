#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for o in ${OPTS:-"reserve_adaptive=0" "reserve_adaptive=1,reserve_extra=2" "reserve_adaptive=1,reserve_extra=4" "reserve_adaptive=1,reserve_extra=6" "reserve_adaptive=1,reserve_extra=8" "reserve_adaptive=1,reserve_extra=4,reserve_min=12"}; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 > gpurun_out/rv_$o.txt 2>&1; head -1 gpurun_out/rv_$o.txt; tail -1 gpurun_out/rv_$o.txt
done
