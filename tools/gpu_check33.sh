#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mixed.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "mixed or bf16 or potrs or leaf" > gpurun_out/pytest_mixed.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mixed.log
tail -4 gpurun_out/pytest_mixed.log
timeout 600 python tools/bench_mixed.py 32768 1024 > gpurun_out/mixed.log 2>&1; echo "rc=$?" >> gpurun_out/mixed.log
timeout 600 python tools/prof_mixed.py 32768 1024 >> gpurun_out/mixed.log 2>&1; echo "rc=$?" >> gpurun_out/mixed.log
cat gpurun_out/mixed.log | tail -8
