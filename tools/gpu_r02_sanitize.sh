#!/bin/bash
# Round-2 GPU call: headline parity tests + compute-sanitizer on every kernel family.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; }
timeout 900 python -m pytest tests/test_headline_parity.py -x -q -m gpu > gpurun_out/headline.log 2>&1; echo "headline rc=$?"
tail -3 gpurun_out/headline.log
CASES="${CASES:-tma_gemm cpasync_gemm chol bf16 tf32 lu qr ltlt contract}"
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tool}_${c}.log | tail -1)"
  done
done
