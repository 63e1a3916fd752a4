#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
rm -f gpurun_out/trees.log
for spec in "1024 128" "2048 128" "2048 256" "3072 128" "4096 128"; do set -- $spec; bs=$1; ib=$2
T="{\"op\":\"cholesky\",\"variant\":3,\"bs\":$bs,\"kernel\":{\"kc\":$bs},\"child\":{\"op\":\"cholesky\",\"variant\":3,\"bs\":$ib,\"kernel\":{\"kc\":$ib},\"child\":{\"op\":\"cholesky\",\"variant\":\"unblocked3\"}}}"
echo "bs=$bs inner=$ib $(timeout 300 python bench.py --no-cpu --no-e2e --no-roofline --steps 2 --warmup 3 --tree "$T" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["value"], d["ms_per_step"])')" >> gpurun_out/trees.log
done
cat gpurun_out/trees.log
timeout 300 python tools/timeline.py 32768 > gpurun_out/timeline.log 2>&1; tail -14 gpurun_out/timeline.log
python tools/prof_chol.py chol 16384 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_16k.csv python tools/prof_chol.py chol 16384 > gpurun_out/ncu_launch.log 2>&1
