#!/bin/bash
# Round-2 profiling pass: full bench line, reference arm, ncu launch list of the
# bench command, one full ncu capture of the dominant kernel (step-0 trailing
# SYRK), the NCCL path at n=32768 and at the C3 size on one GPU.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-side --no-e2e --no-roofline > gpurun_out/r02_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/prof_chol.py syrk 30720 2048 > gpurun_out/r02_syrk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_tma -s 2 -c 1 -o gpurun_out/r02_syrk_full \
    python tools/prof_chol.py syrk 30720 2048 > gpurun_out/r02_ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/r02_syrk_full.ncu-rep --page raw --csv > gpurun_out/r02_syrk_raw.csv 2>/dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29621 \
    bench.py --dist --steps 3 --warmup 3 > gpurun_out/r02_dist1.json 2> gpurun_out/r02_dist1.err; echo "dist rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29622 \
    bench.py --dist --order 131072 --steps 1 --warmup 1 --no-e2e > gpurun_out/r02_dist_c3.json 2> gpurun_out/r02_dist_c3.err; echo "dist c3 rc=$?"
tail -c 600 gpurun_out/r02_bench.json
