#!/bin/bash
# fused diagonal factor parity incl. fused_diag=2 failure cases (bounded: a hang is a bug, not a wait)
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_diag" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_mixed.py -x -q -m gpu -k "npd_pivot" 2>&1 | tail -3
