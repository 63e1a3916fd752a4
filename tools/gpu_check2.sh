#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for a in "tma=1" "tma=0"; do timeout 120 python tools/prof_chol.py syrk 16384 1024 $a >> gpurun_out/syrk_cmp.log 2>&1; done
timeout 120 python tools/prof_chol.py syrk 31744 1024 >> gpurun_out/syrk_cmp.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --no-cpu --no-e2e --no-roofline --n 16384 > gpurun_out/bench16k.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/syrk_cmp.log; tail -2 gpurun_out/bench.log | cut -c1-1500; cut -c1-400 gpurun_out/bench16k.log
