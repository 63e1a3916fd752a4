#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/prof_chol.py syrk 16384 1024 > gpurun_out/syrk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_tma -s 2 -c 1 -o gpurun_out/syrk_tma_full python tools/prof_chol.py syrk 16384 1024 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/syrk_plain.log; tail -2 gpurun_out/ncu_full.log
