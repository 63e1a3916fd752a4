#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "half_width or variants or red_fold or persist or reserv" 2>&1 | tail -2
for o in tma_stagger=0 tma_stagger=1; do
  echo "$o: $(python tools/prof_chol.py syrk 30720 2048 $o 2>/dev/null | tail -1)"
done
for o in ${OPTS:-"tma_stagger=0" "tma_stagger=1"}; do
  BF_OPTS=$o timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-side 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$o', d['ms_per_step'], d['step_ms'])"
done
