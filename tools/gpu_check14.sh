#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/trees.log
for bs in 512 768 1024 1536 2048; do for ib in 64 128; do
T="{\"op\":\"cholesky\",\"variant\":3,\"bs\":$bs,\"kernel\":{\"kc\":$bs},\"child\":{\"op\":\"cholesky\",\"variant\":3,\"bs\":$ib,\"kernel\":{\"kc\":$ib},\"child\":{\"op\":\"cholesky\",\"variant\":\"unblocked3\"}}}"
echo "bs=$bs inner=$ib $(timeout 300 python bench.py --no-cpu --no-e2e --no-roofline --steps 2 --warmup 3 --tree "$T" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["value"], d["ms_per_step"])')" >> gpurun_out/trees.log
done; done
cat gpurun_out/trees.log
