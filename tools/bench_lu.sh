#!/bin/bash
# LU timings through the CLI (median of 3 after a warm-up), several trees
for n in 8192 16384; do
  for t in "1024,128,32" "512,64,16" "1024,256,64,16" "2048,256,32"; do
    IFS=',' read -ra L <<< "$t"
    doc='{"op":"lu","variant":"unblocked"}'
    for ((i=${#L[@]}-1; i>=0; i--)); do doc="{\"op\":\"lu\",\"variant\":\"blocked\",\"bs\":${L[$i]},\"child\":$doc}"; done
    echo "$doc" > /tmp/lu_tree.json
    timeout 600 python -m paper_2604_07311_b200 bench --op lu --n $n --tree /tmp/lu_tree.json | tail -1
  done
done
