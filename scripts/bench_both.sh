#!/bin/bash
# Both bench arms back to back, as the driver runs them (reference first).
# usage: scripts/bench_both.sh <tag> [extra bench args]
tag=${1:-try}; shift
mkdir -p gpurun_out
( time timeout 1700 python bench.py --impl reference "$@" ) > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
( time timeout 1700 python bench.py "$@" ) > gpurun_out/bench_ours_$tag.json 2> gpurun_out/bench_ours_$tag.err
