#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/syrk_var.log
for g in 4 8 16 32; do for v in 0 2; do echo "group=$g variant=$v" >> gpurun_out/syrk_var.log; timeout 120 python tools/prof_chol.py syrk 16384 1024 tma_variant=$v group=$g >> gpurun_out/syrk_var.log 2>&1; done; done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/prof_chol.py chol 16384 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_16k.csv python tools/prof_chol.py chol 16384 > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/syrk_var.log; tail -3 gpurun_out/pytest_gpu.log
