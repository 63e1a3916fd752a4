#!/bin/bash
# grouped trailing update of the NCCL driver: tests, 1x1 timing A/B, C2 regression check
cd "$(dirname "$0")/.."
[ -n "$SKIP_TESTS" ] || timeout 900 python -m pytest tests/test_dist_native.py -x -q -m gpu 2>&1 | tail -3
for o in ${OPTS:-"grouped=0" "grouped=1" "grouped=1;reserve_strided=1"}; do
  d=${o%%;*}; b=""; [ "$d" != "$o" ] && b=${o#*;}
  BF_DIST_OPTS=$d BF_OPTS=$b timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --dist --steps 3 --warmup 2 --no-e2e 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$o', d['ms_per_step'], d['step_ms'])"
done
[ -n "$SKIP_C2" ] || timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'], d['value'])"
