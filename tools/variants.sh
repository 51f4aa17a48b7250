#!/bin/bash
# On the GPU box: time bench.py (config 3 loop) for every lib_v/<variant>/libfpm_b200.so,
# appending "<variant> loop_ms frac sm_mhz" lines to gpurun_out/variants.txt.
# Usage: tools/variants.sh [bench args...]; restores the in-tree library afterwards.
set -u
cp paper_2203_02507_b200/lib/libfpm_b200.so /tmp/libfpm_b200.so.keep
for d in lib_v/*/; do
  v=$(basename "$d")
  cp "$d/libfpm_b200.so" paper_2203_02507_b200/lib/libfpm_b200.so
  timeout 600 python bench.py --no-cpu --no-e2e "$@" > "gpurun_out/bench_$v.log" 2>&1
  python - "$v" <<'PY' >> gpurun_out/variants.txt
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{v}.log").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(v, round(r["loop_ms"], 3), round(r["frac"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(v, "failed", e)
PY
done
cp /tmp/libfpm_b200.so.keep paper_2203_02507_b200/lib/libfpm_b200.so
