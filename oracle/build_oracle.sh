#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY: compile the C restatement of the reference kernels
# (oracle/kernels.c) into oracle/_build/liboracle.so.  -ffp-contract=off keeps
# every a*b+c as two roundings, like the reference's Cython build (gcc -O2,
# baseline x86-64, which has no FMA).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
mkdir -p "$HERE/_build"
gcc -O2 -ffp-contract=off -fPIC -shared -std=c99 "$HERE/kernels.c" -o "$HERE/_build/liboracle.so.tmp" -lm
mv "$HERE/_build/liboracle.so.tmp" "$HERE/_build/liboracle.so"
