#!/bin/bash
# C4: doubling inverse after the (fused) diagonal factor vs the trailing right solve
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_mixed.py -x -q -m gpu 2>&1 | tail -2
for o in mixed_inverse=0 mixed_inverse=1 mixed_inverse=1,mixed_reserve=48 mixed_inverse=1,mixed_reserve=24 mixed_inverse=0 mixed_inverse=1; do
  BF_OPTS=$o timeout 300 python tools/bench_mixed.py 32768 2048 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$o', d['matrix'], d['factor_ms'], d['refine_ms'], d['posv_ms'], d['iterations'], '%.2e' % d['fwd_err_vs_fp64'])"
done
BF_OPTS=mixed_inverse=1 python tools/prof_mixed_chain.py 32768 2048
