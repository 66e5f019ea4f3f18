#!/bin/bash
# A/B of the prebuilt libaqp variants in build/variants/: small-solve latency and C5 pass times
for so in build/variants/*.so; do
  cp $so paper_2602_23967_b200/libaqp.so
  echo "== $so"
  python scripts/c1_time.py
  python scripts/bench_configs.py c5 --windows 2 --warmup 1 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['inner_per_s'], {k: v['us'] for k, v in d['kernels'].items()})"
done
