#!/bin/bash
# Same-box A/B of two builds of the library (BF_LIB_PATH), alternating runs of the n=32768 timeline tool.
OLD=${1:-tools/_ab/lib_old.so}
for r in 1 2; do
  BF_LIB_PATH=$OLD timeout 300 python tools/timeline.py 32768 | grep opts | sed "s/^/old /"
  timeout 300 python tools/timeline.py 32768 | grep opts | sed "s/^/new /"
done
if [ -n "$AB_CONTRACT" ]; then
  BF_LIB_PATH=$OLD timeout 300 python tools/bench_contract.py 128 | sed "s/^/old /"
  timeout 300 python tools/bench_contract.py 128 | sed "s/^/new /"
fi
