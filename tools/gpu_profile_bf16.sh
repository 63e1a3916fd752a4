#!/bin/bash
mkdir -p gpurun_out
python tools/bench_bf16.py > gpurun_out/bf16_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:gemm_bf16_tc -s 7 -c 1 -o gpurun_out/bf16_full python tools/bench_bf16.py > gpurun_out/bf16_ncu.log 2>&1
python tools/bench_mixed.py 32768 1024 > gpurun_out/mixed_plain.log 2>&1
cat gpurun_out/bf16_plain.log gpurun_out/mixed_plain.log; tail -2 gpurun_out/bf16_ncu.log
