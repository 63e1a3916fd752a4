#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -x -p no:cacheprovider -m gpu > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_all.log
tail -3 gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 python tools/bench_mixed.py 32768 1024 > gpurun_out/mixed.log 2>&1; cat gpurun_out/mixed.log
