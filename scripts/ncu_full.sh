#!/bin/bash
# full ncu capture of the hot kernels of a short eager C2 run (one GPU, not a bench number)
export AQP_EAGER=1
OUT=${1:-gpurun_out/prof}
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:OpGrad<\(bool\)0>|OpStep|OpP2|OpP1Bb' -s 40 -c 4 -o $OUT python scripts/prof_c2.py 64
