#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_mixed.py -x -q -m gpu 2>&1 | tail -2
for r in 1 2 3; do timeout 300 python tools/bench_mixed.py 32768 2048 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['matrix'], d['factor_ms'], d['refine_ms'], d['posv_ms'], d['iterations'])"; done
