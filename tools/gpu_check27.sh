#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:trsm_warp_right -s 10 -c 1 -o gpurun_out/trsm_warp python tools/prof_diag.py 1024 1 > gpurun_out/ncu_tw.log 2>&1
tail -2 gpurun_out/ncu_tw.log
