#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/prof_diag.py 2048 5
python tools/prof_diag.py 1024 5
python tools/prof_trsm.py 30720 2048 3
python tools/timeline.py 32768
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag_launches.csv python tools/prof_diag.py 2048 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/trsm_launches.csv python tools/prof_trsm.py 30720 2048 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/diag_launches.csv | head -12
python tools/launch_summary.py gpurun_out/trsm_launches.csv | head -12
