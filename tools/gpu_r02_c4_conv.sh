#!/bin/bash
# C4: A21's bf16 copy beside the diagonal chain (mixed_conv_early) on/off
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_mixed.py -x -q -m gpu 2>&1 | tail -2
for o in mixed_conv_early=0 mixed_conv_early=1 mixed_conv_early=0 mixed_conv_early=1; do
  BF_OPTS=$o timeout 300 python tools/bench_mixed.py 32768 2048 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$o', d['matrix'], d['factor_ms'], d['refine_ms'], d['posv_ms'], d['iterations'], '%.2e' % d['fwd_err_vs_fp64'])"
done
