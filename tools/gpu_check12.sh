#!/bin/bash
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/repro_c292.py c292 > gpurun_out/bisect.log 2>&1
grep -E "match|Error" gpurun_out/bisect.log | tail -2
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e --no-roofline --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
python tools/prof_chol.py chol 16384 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_16k.csv python tools/prof_chol.py chol 16384 > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cut -c1-300 gpurun_out/bench.log
