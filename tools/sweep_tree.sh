#!/bin/bash
# Root/inner block-size sweep of the FP64 bench tree (plain runs, no side measurements).
for rb in 1024 1536 2048 3072; do
  for ib in 64 128 256; do
    t="{\"op\":\"cholesky\",\"variant\":3,\"bs\":$rb,\"kernel\":{\"kc\":$rb},\"child\":{\"op\":\"cholesky\",\"variant\":3,\"bs\":$ib,\"kernel\":{\"kc\":$ib},\"child\":{\"op\":\"cholesky\",\"variant\":\"unblocked3\"}}}"
    if [ $ib -gt 128 ]; then
      t="{\"op\":\"cholesky\",\"variant\":3,\"bs\":$rb,\"kernel\":{\"kc\":$rb},\"child\":{\"op\":\"cholesky\",\"variant\":3,\"bs\":$ib,\"kernel\":{\"kc\":$ib},\"child\":{\"op\":\"cholesky\",\"variant\":3,\"bs\":128,\"kernel\":{\"kc\":128},\"child\":{\"op\":\"cholesky\",\"variant\":\"unblocked3\"}}}}"
    fi
    r=$(timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-side --no-e2e --no-roofline --tree "$t" 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])" 2>&1)
    echo "root $rb inner $ib: $r"
  done
done
