#!/bin/bash
# potrs float4 streams + warp-per-column partial reduction: tests, refinement pieces A/B, C4 end to end
mkdir -p gpurun_out
python -m pytest tests/test_mixed.py -x -q -m gpu 2>&1 | tail -5
for o in potrs_vec=0 potrs_vec=1 potrs_vec=0 potrs_vec=1; do BF_OPTS=$o python tools/prof_refine.py 32768 2048; done
for o in potrs_vec=1; do BF_OPTS=$o python tools/bench_mixed.py 32768 2048; done
python bench.py --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], json.dumps(d.get('side_workloads',{}).get('c4_mixed_posv')))"
