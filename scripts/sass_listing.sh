#!/bin/bash
# SASS listing of every kernel in libaqp.so (instruction lines only, no
# encodings) -> profiles/sass_libaqp_<tag>.txt.gz, plus a per-kernel resource
# table (registers, stack, shared memory) -> profiles/kernel_resources_<tag>.txt
TAG=${1:-r01}
cd "$(dirname "$0")/.."
cuobjdump -sass paper_2602_23967_b200/libaqp.so | grep -v '^\s*/\* 0x' | sed 's#\s*/\* 0x[0-9a-f]* \*/##' \
  | gzip -9 > profiles/sass_libaqp_$TAG.txt.gz
python - "$TAG" <<'PY'
import subprocess, re, sys
out = subprocess.run(["cuobjdump", "-res-usage", "paper_2602_23967_b200/libaqp.so"], capture_output=True, text=True).stdout.splitlines()
rows = set()
for i, l in enumerate(out):
    m = re.match(r"\s*Function (\S+):", l)
    if m and i + 1 < len(out):
        rows.add((subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip(), out[i + 1].strip()))
with open(f"profiles/kernel_resources_{sys.argv[1]}.txt", "w") as f:
    f.write("# cuobjdump -res-usage (sm_100a): registers / stack / smem of every kernel\n")
    for n, r in sorted(rows):
        f.write(f"{r:90s} {n}\n")
PY
ls -la profiles/sass_libaqp_$TAG.txt.gz profiles/kernel_resources_$TAG.txt
