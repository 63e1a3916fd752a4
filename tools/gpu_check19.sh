#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/bench_contract.py 48 64 128 > gpurun_out/contract.log 2>&1
cat gpurun_out/contract.log
