#!/bin/bash
mkdir -p gpurun_out
python tools/prof_chol.py syrk 16384 1024 > gpurun_out/syrk_plain.log 2>&1 && \
python tools/prof_chol.py chol 16384 > gpurun_out/chol_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_16k.csv python tools/prof_chol.py chol 16384 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 2 -c 1 -o gpurun_out/syrk_full python tools/prof_chol.py syrk 16384 1024 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/syrk_plain.log gpurun_out/ncu_launch.log gpurun_out/ncu_full.log
