#!/bin/bash
# Round-end evidence: default bench line, its ncu launch list (after the plain
# run exited 0), and one ncu --set full capture of the trailing SYRK launch the
# bench's roofline quotes (step 0: n_k=30720, K=bs=2048).
mkdir -p gpurun_out
python bench.py > gpurun_out/fz_bench.json 2> gpurun_out/fz_bench.err; echo "bench rc $?"; cat gpurun_out/fz_bench.json
python bench.py --steps 2 --warmup 3 --no-cpu --no-side --no-e2e > gpurun_out/fz_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fz_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-side --no-e2e > gpurun_out/fz_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/fz_launches.csv 100 --skip-first > gpurun_out/fz_launch_summary.txt 2>&1
head -8 gpurun_out/fz_launch_summary.txt
python tools/prof_chol.py syrk 30720 2048 > gpurun_out/fz_syrk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_tma -s 2 -c 1 -o gpurun_out/fz_syrk \
    python tools/prof_chol.py syrk 30720 2048 > gpurun_out/fz_syrk_ncu.log 2>&1; echo "syrk ncu rc $?"; cat gpurun_out/fz_syrk_plain.log
