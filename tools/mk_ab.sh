#!/bin/bash
# Build the library as of git HEAD into tools/_ab/lib_old.so (for tools/gpu_ab.sh), then rebuild the working tree.
set -e
cd "$(dirname "$0")/.."
git stash push -q -- paper_2604_07311_b200/csrc include
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p tools/_ab && cp paper_2604_07311_b200/_lib/libblockfam_b200.so tools/_ab/lib_old.so
git stash pop -q
python -c "import __graft_entry__ as g; g.build()" > /dev/null
