#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/bench_mixed.py 8192 1024 > gpurun_out/mixed.log 2>&1; echo "rc=$?" >> gpurun_out/mixed.log
timeout 600 python tools/bench_mixed.py 32768 1024 >> gpurun_out/mixed.log 2>&1; echo "rc=$?" >> gpurun_out/mixed.log
cat gpurun_out/mixed.log | tail -20
