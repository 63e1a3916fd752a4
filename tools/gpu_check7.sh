#!/bin/bash
mkdir -p gpurun_out
./tools/loop_probe > gpurun_out/loop_probe.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/prof_chol.py syrk 16384 1024 tma_variant=2 > gpurun_out/syrk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_tma -s 2 -c 1 -o gpurun_out/syrk_tma_v2 python tools/prof_chol.py syrk 16384 1024 tma_variant=2 > gpurun_out/ncu_full.log 2>&1
python tools/prof_chol.py chol 16384 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_16k.csv python tools/prof_chol.py chol 16384 > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/loop_probe.log; tail -3 gpurun_out/pytest_gpu.log
