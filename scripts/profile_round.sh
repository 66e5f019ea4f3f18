#!/bin/bash
# Profiling evidence for profiles/ (run on the GPU box, one GPU; never a bench number):
#  1. launch list of one C2 certification window (eager mode: ncu cannot
#     profile kernel nodes of graphs that contain conditional nodes)
#  2. ncu --set full of the hot kernels: C2 (BB gradient / step / fold, P1, P2),
#     C5 (gradient, P1, P2), C3 (dense R x, dense R'(R x))
set -x
mkdir -p gpurun_out/ncu
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -f"
AQP_EAGER=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -c 5000 --csv --log-file gpurun_out/launches.csv \
    python scripts/prof_c2.py 64 > gpurun_out/launches_stdout.txt 2>&1
AQP_EAGER=1 $NCU -k 'regex:spmv_op<aqp::OpGrad<\(bool\)0>, \(bool\)1>' -s 20 -c 1 -o gpurun_out/ncu/c2_bb_gradient \
    python scripts/prof_c2.py 64 > gpurun_out/ncu/c2.log 2>&1
AQP_EAGER=1 $NCU -k 'regex:elem_op<aqp::OpStep' -s 20 -c 1 -o gpurun_out/ncu/c2_bb_step \
    python scripts/prof_c2.py 64 >> gpurun_out/ncu/c2.log 2>&1
AQP_EAGER=1 $NCU -k 'regex:fin_ctrl_(op|cl)<aqp::OpGrad<\(bool\)0>' -s 20 -c 1 -o gpurun_out/ncu/c2_bb_fold \
    python scripts/prof_c2.py 64 >> gpurun_out/ncu/c2.log 2>&1
AQP_EAGER=1 $NCU -k 'regex:spmv_op<aqp::OpP1Bb' -s 2 -c 1 -o gpurun_out/ncu/c2_p1 \
    python scripts/prof_c2.py 64 >> gpurun_out/ncu/c2.log 2>&1
AQP_EAGER=1 $NCU -k 'regex:spmv_op<aqp::OpP2' -s 2 -c 1 -o gpurun_out/ncu/c2_p2 \
    python scripts/prof_c2.py 64 >> gpurun_out/ncu/c2.log 2>&1
$NCU -k 'regex:spmv_op<aqp::(OpGrad|OpP1Bb|OpP2)' -c 3 -o gpurun_out/ncu/c5_passes \
    python scripts/prof_kernel.py c5 0,2,3 > gpurun_out/ncu/c5.log 2>&1
$NCU -k 'regex:k_dense_rx\(|k_dense_rtv' -c 2 -o gpurun_out/ncu/c3_dense \
    python scripts/prof_kernel.py c3 6,7 > gpurun_out/ncu/c3.log 2>&1
ls -la gpurun_out gpurun_out/ncu
