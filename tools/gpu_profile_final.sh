#!/bin/bash
# End-of-round profiling: plain bench line, its ncu launch list, and full ncu
# captures of the leaf and fused-TRSM kernels (the panel-chain kernels).
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu --no-side --no-e2e > gpurun_out/fin_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fin_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-side --no-e2e > gpurun_out/fin_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/fin_launches.csv --skip-first > gpurun_out/fin_launch_summary.txt 2>&1
python tools/prof_diag.py 1024 2 > gpurun_out/fin_diag_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:potrf_leaf_blocked -s 2 -c 1 -o gpurun_out/fin_leaf \
    python tools/prof_diag.py 1024 1 > gpurun_out/fin_ncu_leaf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:trsm_warp_right -s 10 -c 1 -o gpurun_out/fin_trsm \
    python tools/prof_diag.py 1024 1 > gpurun_out/fin_ncu_trsm.log 2>&1
tail -1 gpurun_out/fin_plain.log | cut -c1-200; cat gpurun_out/fin_launch_summary.txt; ls gpurun_out/fin_*
