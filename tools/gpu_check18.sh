#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist.py -q -p no:cacheprovider > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist.log
tail -3 gpurun_out/pytest_dist.log
timeout 600 python bench.py --dist --steps 2 --warmup 3 > gpurun_out/bench_dist1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_dist1.log
cut -c1-600 gpurun_out/bench_dist1.log | tail -3
