#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mixed.py -q -x -p no:cacheprovider > gpurun_out/pytest_mixed.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mixed.log
tail -5 gpurun_out/pytest_mixed.log
timeout 600 python tools/bench_mixed.py 32768 1024 > gpurun_out/mixed.log 2>&1; echo "rc=$?" >> gpurun_out/mixed.log
timeout 600 python tools/prof_mixed.py 32768 1024 >> gpurun_out/mixed.log 2>&1; echo "rc=$?" >> gpurun_out/mixed.log
cat gpurun_out/mixed.log | tail -20
