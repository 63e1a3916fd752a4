#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/syrk_k.log
for bs in 256 512 1024 2048 4096; do timeout 120 python tools/prof_chol.py syrk 16384 $bs >> gpurun_out/syrk_k.log 2>&1; done
for t in 0 4; do echo "tpc=$t" >> gpurun_out/syrk_k.log; for bs in 256 1024; do timeout 120 python tools/prof_chol.py syrk 16384 $bs tiles_per_cta=$t >> gpurun_out/syrk_k.log 2>&1; done; done
cat gpurun_out/syrk_k.log
