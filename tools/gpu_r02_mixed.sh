#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_mixed.py tests/test_f32_tc.py -x -q -m gpu 2>&1 | tail -2
for o in ${OPTS:-"mixed_fast_inverse=0" "mixed_fast_inverse=1" "mixed_fast_inverse=1,mixed_reserve=24" "mixed_fast_inverse=1,mixed_reserve=48"}; do
  BF_OPTS=$o STEP_TOL=1e-11 timeout 300 python tools/bench_mixed.py 32768 1024 2>&1 | head -1 | cut -c1-330
done
python tools/prof_mixed_chain.py 2>&1 | tail -1
