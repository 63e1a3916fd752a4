#!/bin/bash
# ncu full captures of the C5 TMEM-fold kernel: plain facade (abij,cdij) vs mode groups (aibj,cidj)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --set full --clock-control none --kernel-name-base demangled -k "regex:\(int\)3, \(bool\)1, \(bool\)0" -s 1 -c 1 \
    -o gpurun_out/c5_plain python tools/c5_perm.py 128 > gpurun_out/c5_plain_ncu.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --kernel-name-base demangled -k "regex:\(int\)3, \(bool\)1, \(bool\)1" -s 1 -c 1 \
    -o gpurun_out/c5_modes python tools/c5_perm.py 128 > gpurun_out/c5_modes_ncu.log 2>&1; echo "modes rc=$?"
for f in c5_plain c5_modes; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; done
ls -la gpurun_out/c5_*
