#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_mixed.py tests/test_f32_tc.py -x -q -m gpu 2>&1 | tail -2
BF_OPTS=mixed_reserve=32 timeout 300 python tools/bench_mixed.py 32768 1024 2>&1 | head -2
timeout 600 python tools/sweep_mixed_diag.py 32768 1024 2>&1
