#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mixed.py -q -x -p no:cacheprovider > gpurun_out/pytest_mixed.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mixed.log
tail -25 gpurun_out/pytest_mixed.log
