#!/bin/bash
# full ncu capture of the three level-0 hot kernels of one metric sort (run under gpurun)
# usage: tools/ncu_hot.sh <out-name> [p] [s]
set -e
OUT=${1:-prof}
shift || true
python tools/prof_one.py "$@" > gpurun_out/${OUT}_plain.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${NCU_K:-k_(hist|scatter|scatter_wc|bucket_sort)<\(int\)0}" -c 4 -o gpurun_out/${OUT} \
    python tools/prof_one.py "$@" > gpurun_out/${OUT}_ncu.log 2>&1
tail -3 gpurun_out/${OUT}_ncu.log
