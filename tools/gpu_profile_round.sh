#!/bin/bash
# Round profiling pass: plain bench, its ncu launch list, and one full ncu
# capture of the dominant kernel (the step-0 trailing SYRK of the bench tree).
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r01_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r01_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r01_ncu_launch.log 2>&1
python tools/prof_chol.py syrk 30720 2048 > gpurun_out/r01_syrk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_tma -s 2 -c 1 -o gpurun_out/r01_syrk_full \
    python tools/prof_chol.py syrk 30720 2048 > gpurun_out/r01_ncu_full.log 2>&1
tail -1 gpurun_out/r01_plain.log | cut -c1-200; tail -2 gpurun_out/r01_ncu_full.log; cat gpurun_out/r01_syrk_plain.log
