#!/bin/bash
# time the hot kernels for each prebuilt libaqp variant in build/variants/
for so in build/variants/*.so; do
  cp $so paper_2602_23967_b200/libaqp.so
  echo "== $so"; AQP_STAGED_MIN=1e9 python scripts/kern_times.py
done
