#!/bin/bash
# fused diagonal factor: parity test, then the 2048 factor alone with fused_diag 0/1 and grid sizes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k fused_diag 2>&1 | tail -3
for o in fused_diag=0 fused_diag=1 fused_diag=1,fused_diag_ctas=16 fused_diag=1,fused_diag_ctas=32 fused_diag=1,fused_diag_ctas=64; do
  echo "== $o"; BF_OPTS=$o timeout 120 python tools/prof_diag.py 2048 3 | sed 's/tree=.*}}: ms/ms/'
done
