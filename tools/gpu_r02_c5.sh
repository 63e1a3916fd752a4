#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_cuda_golden.py tests/test_headline_parity.py tests/test_gpu_parity.py -x -q -m gpu -k "contract or K64 or K128 or tma or gemm" 2>&1 | tail -2
timeout 600 python tools/c5_tmem.py 128 3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_dmma_tma_kernel -c 2 python tools/c5_tmem.py 128 1 1 > gpurun_out/c5_ncu.txt 2>&1; echo ncu rc=$?
grep -E "gemm_dmma|duration|dram__|hit_rate|fp64" gpurun_out/c5_ncu.txt | head -20
