#!/bin/bash
for so in build/variants/*.so; do
  cp $so paper_2602_23967_b200/libaqp.so
  echo "== $so"
  AQP_STAGED_MIN=1e9 python scripts/kern_times.py | python -c "
import sys, json; d = json.loads(sys.stdin.read()); print({k: v['us'] for k, v in d.items()})"
  python scripts/bench_configs.py c2 --windows 4 --warmup 1 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], 'inner/s', d['inner_per_s'])"
done
