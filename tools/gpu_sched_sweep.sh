#!/bin/bash
# Schedule-option sweep of the n=32768 factorization (timeline plain timings)
# plus one ncu --set full capture of the C5 contraction GEMM.
mkdir -p gpurun_out
for o in "" pipeline_first=2 pipeline_first=4 pipeline_first=8 tail_reserve=8 tail_reserve=24 tail_reserve=32; do
  BF_OPTS=$o timeout 300 python tools/timeline.py 32768 > gpurun_out/ss_$o.txt 2>&1
  head -1 gpurun_out/ss_$o.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_tma -c 1 -o gpurun_out/contract_red \
  python tools/prof_contract_one.py 128 > gpurun_out/contract_red_ncu.log 2>&1; echo "ncu rc $?"
