#!/bin/bash
# time the hot kernels (C2, stand-alone, L2 flushed) and a short C2 window run
# for each prebuilt libaqp variant in build/variants/
for so in build/variants/*.so; do
  cp $so paper_2602_23967_b200/libaqp.so
  echo "== $so"; AQP_STAGED_MIN=1e9 python scripts/kern_times.py
  python scripts/bench_configs.py c2 --windows 4 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('window inner/s', d['inner_per_s'])"
done
