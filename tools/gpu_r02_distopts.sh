#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for o in "fan=3" "fan=0" "fan=1" "fan=3,reserve=0" "fan=0,reserve=24"; do
  BF_DIST_OPTS=$o timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --dist --steps 3 --warmup 2 --no-e2e 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$o', d['ms_per_step'], d['step_ms'])"
done
for t in '{"op":"cholesky","variant":3,"bs":1024,"kernel":{"kc":1024},"child":{"op":"cholesky","variant":3,"bs":128,"kernel":{"kc":128},"child":{"op":"cholesky","variant":"unblocked3"}}}'; do
  BF_DIST_OPTS=fan=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --dist --steps 3 --warmup 2 --no-e2e --tree "$t" 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('nb1024 fan0', d['ms_per_step'], d['step_ms'])"
done
