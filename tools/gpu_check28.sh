#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused_trsm" > gpurun_out/pytest_tw.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tw.log
tail -2 gpurun_out/pytest_tw.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag_launches.csv python tools/prof_diag.py 1024 1 > gpurun_out/diag_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/diag_launches.csv 2>&1 | head -5
