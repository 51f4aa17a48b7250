#!/bin/bash
# On the GPU box: bench.py config 5 per lib_v/<variant>/libfpm_b200.so (4-CTA clusters),
# printing "<variant> step_ms loop_ms frac" into gpurun_out/c5_variants.txt.
cp paper_2203_02507_b200/lib/libfpm_b200.so /tmp/keep.so
for d in lib_v/*/; do
  v=$(basename "$d")
  cp "$d/libfpm_b200.so" paper_2203_02507_b200/lib/libfpm_b200.so
  timeout 600 python bench.py --config 5 --steps 3 --no-cpu --no-e2e "$@" > gpurun_out/c5_$v.log 2>&1
  python - $v <<'PY' >> gpurun_out/c5_variants.txt
import json,sys
v=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/c5_{v}.log").read().strip().splitlines()[-1]); r=d["roofline"]
    print(v, round(d["ms_per_step"],1), round(r["loop_ms"],1), round(r["frac"],4))
except Exception as e: print(v, "failed", open(f"gpurun_out/c5_{v}.log").read()[-300:])
PY
done
cp /tmp/keep.so paper_2203_02507_b200/lib/libfpm_b200.so
