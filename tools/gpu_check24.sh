#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/prof_diag.py 1024 3 > gpurun_out/diag.log 2>&1; echo "rc=$?" >> gpurun_out/diag.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag_launches.csv python tools/prof_diag.py 1024 1 > gpurun_out/diag_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/diag_launches.csv >> gpurun_out/diag.log 2>&1
cat gpurun_out/diag.log
