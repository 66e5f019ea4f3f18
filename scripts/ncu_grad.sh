#!/bin/bash
# ncu capture of the stand-alone BB gradient pass (kernel timing path, no graph)
OUT=${1:-gpurun_out/prof_grad}
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:spmv_op<aqp::OpGrad<\(bool\)0>' -s 3 -c 1 -o $OUT python scripts/kern_times.py
