#!/bin/bash
# A/B of SELL-32 copies for uniform plans (AQP_SELL=1 default vs 0) and of the
# vectorised tile staging (prebuilt variants in build/variants/): C2 hot
# kernels, a C2 window, small solves, C5 passes
for sell in 1 0; do
  echo "== AQP_SELL=$sell"
  AQP_SELL=$sell python scripts/kern_times.py
  AQP_SELL=$sell python scripts/bench_configs.py c2 c5 --windows 2 --warmup 1 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], 'inner/s', d['inner_per_s'], {k: v['us'] for k, v in d['kernels'].items()})"
done
