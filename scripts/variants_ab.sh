#!/bin/bash
# A/B the prebuilt libaqp variants (scripts/build_variants.sh) on stand-alone
# hot-kernel timings: C5-shaped n=m=1e7 (w=5000) and C2.  One JSON line per run.
#   scripts/variants_ab.sh [variant ...]     (default: every build/variants/*.so)
cd "$(dirname "$0")/.."
cp paper_2602_23967_b200/libaqp.so /tmp/libaqp_orig.so
vs="$@"
[ -z "$vs" ] && vs=$(ls build/variants/*.so | xargs -n1 basename | sed 's/\.so$//')
for v in $vs; do
  cp build/variants/$v.so paper_2602_23967_b200/libaqp.so
  echo "== $v"
  timeout 300 python scripts/c5_kernels.py --n 1e7 "" 2>&1 | tail -1
  timeout 300 python scripts/c5_kernels.py --spec c2 "" 2>&1 | tail -1
done
cp /tmp/libaqp_orig.so paper_2602_23967_b200/libaqp.so
