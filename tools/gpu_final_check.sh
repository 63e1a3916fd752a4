#!/bin/bash
# Final round check: full GPU suite + smoke, and LU timings at the DESIGN trees.
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/fx_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/fx_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo '{"op":"lu","variant":"blocked","bs":512,"kernel":{"kc":512},"child":{"op":"lu","variant":"blocked","bs":32,"child":{"op":"lu","variant":"unblocked"}}}' > /tmp/lu16.json
echo '{"op":"lu","variant":"blocked","bs":1024,"kernel":{"kc":1024},"child":{"op":"lu","variant":"blocked","bs":128,"child":{"op":"lu","variant":"blocked","bs":32,"child":{"op":"lu","variant":"unblocked"}}}}' > /tmp/lu32.json
timeout 600 python -m paper_2604_07311_b200 bench --op lu --n 16384 --tree /tmp/lu16.json 2>&1 | tail -2
timeout 900 python -m paper_2604_07311_b200 bench --op lu --n 32768 --tree /tmp/lu32.json 2>&1 | tail -2
