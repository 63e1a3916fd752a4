#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
python tools/prof_chol.py chol 2048 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:potrf_leaf -s 3 -c 1 -o gpurun_out/leaf_full python tools/prof_chol.py chol 2048 > gpurun_out/ncu_leaf.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | cut -c1-400
