#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:trsm_small_right_kernel -s 3 -c 1 -o gpurun_out/trsm_small python tools/prof_diag.py 1024 1 > gpurun_out/ncu_trsm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:potrf_leaf_v3 -s 3 -c 1 -o gpurun_out/leaf_v3 python tools/prof_diag.py 1024 1 >> gpurun_out/ncu_trsm.log 2>&1
tail -3 gpurun_out/ncu_trsm.log; ls -la gpurun_out/*.ncu-rep
