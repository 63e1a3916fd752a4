#!/bin/bash
# ncu --set full of the kernels changed late in round 2: the cooperative refinement solve and the fused
# diagonal factor (each command exits 0 without ncu first)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/prof_refine.py 32768 2048 > /dev/null 2>&1 && echo refine ok
python tools/prof_diag.py 2048 2 > /dev/null 2>&1 && echo diag ok
timeout 900 ncu --set full --clock-control none --import-source on -k regex:potrs_coop -s 2 -c 1 \
  -o gpurun_out/potrs_coop python tools/prof_refine.py 32768 2048 > gpurun_out/ncu_potrs.log 2>&1; echo "ncu potrs rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:potrf_diag_fused -s 1 -c 1 \
  -o gpurun_out/diag_fused python tools/prof_diag.py 2048 2 > gpurun_out/ncu_diag.log 2>&1; echo "ncu diag rc=$?"
ls -la gpurun_out/*.ncu-rep
