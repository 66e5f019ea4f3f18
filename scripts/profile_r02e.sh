#!/bin/bash
# Round-2 (ring path) profiling evidence (GPU box, one GPU; never a bench number):
#  1. the launch list of the bench command itself (eager mode: ncu cannot see the
#     kernel nodes of graphs with conditional nodes), per-launch device time
#  2. ncu --set full of the hot kernels stand-alone: C5 (gradient, step, P1 SELL-P,
#     P2, X, fold) and C2 (gradient, P1, P2)
mkdir -p gpurun_out/ncu
export AQP_BENCH_NO_SECONDARY=1
[ "$1" = "--no-launches" ] || AQP_EAGER=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
    -c 3000 --csv --log-file gpurun_out/launches_r02e.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_r02e_stdout.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -f"
timeout 1200 $NCU -k 'regex:spmv_op<|spmv_sellp_op<|spmv_ring_op<|k_step2|fin_ctrl_cl<|elem_op<aqp::OpXPost' -c 10 -o gpurun_out/ncu/c5_r02e \
    python scripts/prof_kernel.py c5 0,1,2,3,4,5 > gpurun_out/ncu/c5_r02e.log 2>&1
timeout 900 $NCU -k 'regex:spmv_op<|spmv_sellp_op<|spmv_ring_op<|k_step2|fin_ctrl_cl<|elem_op<aqp::OpXPost' -c 10 -o gpurun_out/ncu/c2_r02e \
    python scripts/prof_kernel.py c2 0,1,2,3,4,5 > gpurun_out/ncu/c2_r02e.log 2>&1
ls -la gpurun_out gpurun_out/ncu
