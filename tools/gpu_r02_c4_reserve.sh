#!/bin/bash
# C4: side-chain SM reservation x fused diagonal factor (fused_diag=2 releases the inverse per column)
cd "$(dirname "$0")/.."
for o in mixed_reserve=32,fused_diag=1 mixed_reserve=48,fused_diag=1 mixed_reserve=64,fused_diag=1 \
         mixed_reserve=32,fused_diag=2 mixed_reserve=48,fused_diag=2 mixed_reserve=64,fused_diag=2 mixed_reserve=80,fused_diag=2; do
  BF_OPTS=$o timeout 300 python tools/bench_mixed.py 32768 2048 2>/dev/null | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', d['factor_ms'], d['posv_ms'])"
done
