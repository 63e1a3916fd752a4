#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/syrk_k.log
for bs in 256 1024 4096; do timeout 120 python tools/prof_chol.py syrk 16384 $bs >> gpurun_out/syrk_k.log 2>&1; done
cat gpurun_out/syrk_k.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for bs in 1024 2048; do
T="{\"op\":\"cholesky\",\"variant\":3,\"bs\":$bs,\"kernel\":{\"kc\":$bs},\"child\":{\"op\":\"cholesky\",\"variant\":3,\"bs\":128,\"kernel\":{\"kc\":128},\"child\":{\"op\":\"cholesky\",\"variant\":\"unblocked3\"}}}"
echo "bs=$bs $(timeout 300 python bench.py --no-cpu --no-e2e --no-roofline --steps 2 --warmup 3 --tree "$T" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["value"], d["ms_per_step"])')"
done
