#!/bin/bash
# 128x64 two-CTA-per-SM TMA tiles: bitwise tests, standalone SYRK rate, C2
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "half_width or variants or red_fold or persist" 2>&1 | tail -2
for o in 128 64; do
  echo "tma_bn=$o: $(python tools/prof_chol.py syrk 16384 2048 tma_bn=$o 2>/dev/null | tail -1)"
  echo "tma_bn=$o: $(python tools/prof_chol.py syrk 30720 2048 tma_bn=$o 2>/dev/null | tail -1)"
done
for o in ${OPTS:-"tma_bn=128" "tma_bn=64"}; do
  BF_OPTS=$o timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$o', d['ms_per_step'], d['step_ms'])"
done
