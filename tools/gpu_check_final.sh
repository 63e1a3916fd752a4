#!/bin/bash
# Round-end check: full GPU test suite, smoke, the default bench line, and the
# bench's ncu launch list (after the plain run exited 0).
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/fin_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/fin_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/fin_smoke.log
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc $?"
python bench.py --steps 2 --warmup 3 --no-cpu --no-side --no-e2e > gpurun_out/fin_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fin_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-side --no-e2e > gpurun_out/fin_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/fin_launches.csv 100 --skip-first > gpurun_out/fin_launch_summary.txt 2>&1
cat gpurun_out/fin_launch_summary.txt | head -12
