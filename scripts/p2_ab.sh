#!/bin/bash
for so in build/variants/*.so; do
  cp $so paper_2602_23967_b200/libaqp.so
  echo "== $so"
  python scripts/bench_configs.py c2 c5 --windows 2 --warmup 1 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['inner_per_s'], 'p2', d['kernels']['p2_A_xbar']['us'], 'p1', d['kernels']['p1_At_y']['us'])"
done
