#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2 3; do timeout 120 python tools/prof_chol.py syrk 16384 1024 tma_variant=$v >> gpurun_out/syrk_var.log 2>&1; done
timeout 120 python tools/prof_chol.py syrk 16384 1024 tma=0 >> gpurun_out/syrk_var.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
python tools/prof_chol.py chol 16384 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_16k.csv python tools/prof_chol.py chol 16384 > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/syrk_var.log; tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | cut -c1-300
