#!/bin/bash
# Round-1 late profiles: tf32 GEMM (ncu full, one launch), LU / LTLT / QR launch lists.
mkdir -p gpurun_out
python tools/bench_tf32.py > gpurun_out/tf32_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:gemm_bf16_tc -s 1 -c 1 -o gpurun_out/tf32_full python tools/bench_tf32.py > gpurun_out/tf32_ncu.log 2>&1
python tools/prof_lu.py 16384 512,32 512 > gpurun_out/lu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu_launch.csv python tools/prof_lu.py 16384 512,32 512 > /dev/null 2>&1
python tools/prof_ltlt.py 4096 128 2 > gpurun_out/ltlt_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ltlt_launch.csv python tools/prof_ltlt.py 4096 128 1 > /dev/null 2>&1
python tools/prof_qr.py 8192 4096 128 3 > gpurun_out/qr_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr_launch.csv python tools/prof_qr.py > /dev/null 2>&1
cat gpurun_out/tf32_plain.log gpurun_out/lu_plain.log gpurun_out/ltlt_plain.log gpurun_out/qr_plain.log; tail -2 gpurun_out/tf32_ncu.log
