#!/bin/bash
# 2048 diagonal factor: wall time alone, then the ncu launch list of one factorization
mkdir -p gpurun_out
python tools/prof_diag.py 2048 5
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag_launches.csv \
    python tools/prof_diag.py 2048 1 > gpurun_out/diag_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/diag_launches.csv 2>&1 | head -30
