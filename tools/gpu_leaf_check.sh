#!/bin/bash
# Full GPU suite, the n=32768 timeline, and the leaf launch times of one
# factorization (how many leaves take the exact redo).
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/lf_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/lf_tests.log
timeout 300 python tools/timeline.py 32768 > gpurun_out/lf_timeline.txt 2>&1; head -1 gpurun_out/lf_timeline.txt; tail -1 gpurun_out/lf_timeline.txt
python tools/prof_chol.py chol 32768 > gpurun_out/lf_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf_leaf --csv --log-file gpurun_out/lf_leaf.csv \
    python tools/prof_chol.py chol 32768 > gpurun_out/lf_ncu.log 2>&1; echo "ncu rc $?"
