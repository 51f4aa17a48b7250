#!/bin/bash
# On the GPU box: bench.py config 3 per lib_v/<variant>/libfpm_b200.so, printing
# "<variant> step loop init finalize" (ms) into gpurun_out/variants_phases.txt.
set -u
cp paper_2203_02507_b200/lib/libfpm_b200.so /tmp/libfpm_b200.so.keep
for d in lib_v/*/; do
  v=$(basename "$d")
  cp "$d/libfpm_b200.so" paper_2203_02507_b200/lib/libfpm_b200.so
  timeout 600 python bench.py --no-cpu --no-e2e "$@" > "gpurun_out/bench_$v.log" 2>&1
  python - "$v" <<'PY' >> gpurun_out/variants_phases.txt
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{v}.log").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(v, round(d["ms_per_step"], 3), round(r["loop_ms"], 3), round(r["init_ms"], 3), round(r["finalize_ms"], 3))
except Exception as e:
    print(v, "failed", e)
PY
done
cp /tmp/libfpm_b200.so.keep paper_2203_02507_b200/lib/libfpm_b200.so
