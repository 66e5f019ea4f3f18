#!/bin/bash
# Profiling evidence for profiles/ (run on the GPU box, one GPU):
#  1. launch list of one C2 certification window (eager mode: ncu cannot
#     profile kernel nodes of graphs that contain conditional nodes)
#  2. ncu --set full of the dominant kernel (uniform THREAD-plan BB gradient SpMV)
set -x
export AQP_EAGER=1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -c 5000 --csv --log-file gpurun_out/launches.csv \
    python scripts/prof_c2.py 64 > gpurun_out/launches_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:spmv_op<aqp::OpGrad<\(bool\)0>, \(bool\)1>' -s 20 -c 2 -o gpurun_out/prof_grad \
    python scripts/prof_c2.py 64 > gpurun_out/prof_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:elem_op<aqp::OpStep' -s 20 -c 1 -o gpurun_out/prof_step \
    python scripts/prof_c2.py 64 >> gpurun_out/prof_stdout.txt 2>&1
ls -la gpurun_out
