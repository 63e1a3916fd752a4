#!/bin/bash
# native NCCL driver at N=1 (C2 size), fused diagonal factor on/off, tiles 2048 (N<=2) and 1024 (N>2 tree)
cd "$(dirname "$0")/.."
T1024='{"op": "cholesky", "variant": 3, "bs": 1024, "kernel": {"kc": 1024}, "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128}, "child": {"op": "cholesky", "variant": "unblocked3"}}}'
p=29611
for r in 1 2; do
  for o in fused_diag=0 fused_diag=1; do
    p=$((p+1))
    BF_OPTS=$o timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port $p bench.py --dist --steps 3 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o tiles2048', d['ms_per_step'])"
    p=$((p+1))
    BF_OPTS=$o timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port $p bench.py --dist --steps 3 --warmup 3 --no-e2e --tree "$T1024" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o tiles1024', d['ms_per_step'])"
  done
done
