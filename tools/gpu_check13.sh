#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/timeline.py 32768 > gpurun_out/timeline.log 2>&1
cat gpurun_out/timeline.log
