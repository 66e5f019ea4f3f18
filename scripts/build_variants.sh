#!/bin/bash
# Build libaqp variants (extra -D flags) into build/variants/<name>.so for A/B kernel timing.
#   scripts/build_variants.sh name1 "-DFOO=1" name2 "-DFOO=2" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants build/vobj
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Iinclude"
while [ $# -gt 0 ]; do
  name=$1; defs=$2; shift 2
  objs=""
  for src in aqp_problem aqp_solver aqp_registry aqp_scale aqp_xfer aqp_setup; do
    /usr/local/cuda/bin/nvcc $FL $defs -c paper_2602_23967_b200/csrc/$src.cu -o build/vobj/${name}_$src.o &
    objs="$objs build/vobj/${name}_$src.o"
  done
  wait
  /usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs -o build/variants/$name.so
  echo "built $name ($defs)"
done
