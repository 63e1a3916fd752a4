#!/bin/bash
# Bench-tree sweep under the SM-reservation schedule (plain timings, n=32768).
mkdir -p gpurun_out
leaf='{"op":"cholesky","variant":"unblocked3"}'
lvl() { echo "{\"op\":\"cholesky\",\"variant\":3,\"bs\":$1,\"kernel\":{\"kc\":$1},\"child\":$2}"; }
# SPECS="2048 128;2048 64" overrides the list (';'-separated trees of block sizes)
IFS=';' read -ra specs <<< "${SPECS:-2048 128;2048 64;2048 256 128;2048 512 128;2048 256 64;2048 512 64;1024 128;4096 128;4096 512 128;2048 1024 128}"
for spec in "${specs[@]}"; do
  set -- $spec
  t=$leaf
  for ((i=$#; i>=1; i--)); do t=$(lvl ${!i} "$t"); done
  timeout 300 python tools/timeline.py 32768 "$t" 2>&1 | grep -E "^opts" | sed "s/^/[$spec] /"
done
