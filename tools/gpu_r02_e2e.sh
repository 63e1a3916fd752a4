#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_cuda_golden.py tests/test_headline_parity.py -x -q -m gpu 2>&1 | tail -2
for o in "wavefront=0" "wavefront=1"; do
  BF_OPTS=$o timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-side --no-roofline --e2e-steps 3 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$o', 'dev', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'])"
done
