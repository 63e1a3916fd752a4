#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/tpc.log
for t in 1 2 4 0; do echo "tpc=$t" >> gpurun_out/tpc.log; timeout 120 python tools/prof_chol.py syrk 16384 1024 tiles_per_cta=$t >> gpurun_out/tpc.log 2>&1; timeout 300 python bench.py --no-cpu --no-e2e --no-roofline --steps 2 --warmup 3 --tiles-per-cta $t 2>&1 | cut -c1-200 >> gpurun_out/tpc.log; done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/tpc.log; tail -3 gpurun_out/pytest_gpu.log
