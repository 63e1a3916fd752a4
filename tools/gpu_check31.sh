#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -x -p no:cacheprovider -m gpu > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_all.log
tail -15 gpurun_out/pytest_all.log | grep -v "^$" | tail -6
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag_launches.csv python tools/prof_diag.py 1024 1 > gpurun_out/diag_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/diag_launches.csv 2>&1 | head -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-250
