#!/bin/bash
# Round 2: the native NCCL driver on one GPU (tests + bench --dist at N=1).
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_dist_native.py tests/test_dist.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --dist --steps 3 --warmup 3 --no-e2e > gpurun_out/dist_bench.log 2>&1; echo "dist bench rc=$?"
tail -c 3000 gpurun_out/dist_bench.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-side --no-e2e --no-roofline > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench1.log
