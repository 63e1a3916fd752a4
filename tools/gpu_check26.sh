#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused_trsm" > gpurun_out/pytest_tw.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tw.log
tail -4 gpurun_out/pytest_tw.log
timeout 120 python tools/prof_diag.py 1024 3 > gpurun_out/diag.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag_launches.csv python tools/prof_diag.py 1024 1 > gpurun_out/diag_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/diag_launches.csv >> gpurun_out/diag.log 2>&1
cat gpurun_out/diag.log | head -9
timeout 600 python -m pytest tests/ -q -x -p no:cacheprovider -m gpu > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_all.log
tail -3 gpurun_out/pytest_all.log
timeout 600 python tools/bench_mixed.py 32768 1024 > gpurun_out/mixed.log 2>&1; cat gpurun_out/mixed.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
