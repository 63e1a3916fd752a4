#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "host" 2>&1 | tail -2
for o in "chunked_load=0" "chunked_load=2" "chunked_load=4" "chunked_load=6"; do
  BF_OPTS=$o timeout 600 python tools/timeline_host.py 32768 2>&1 | head -4
done
