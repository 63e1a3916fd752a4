#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2 3; do timeout 120 python tools/prof_chol.py syrk 16384 1024 tma_variant=$v >> gpurun_out/syrk_var.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/syrk_var.log; tail -5 gpurun_out/pytest_gpu.log
