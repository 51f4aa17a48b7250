cp paper_2203_02507_b200/lib/libfpm_b200.so /tmp/keep.so
for v in base db256; do
  cp lib_v/$v/libfpm_b200.so paper_2203_02507_b200/lib/libfpm_b200.so
  for cl in 4 8; do
    FPM_B200_CLUSTER=$cl timeout 600 python bench.py --config 5 --steps 3 --no-cpu --no-e2e > gpurun_out/c5_${v}_$cl.log 2>&1
    python - $v $cl <<'PY'
import json,sys
v,cl=sys.argv[1:]
try:
    d=json.loads(open(f"gpurun_out/c5_{v}_{cl}.log").read().strip().splitlines()[-1]); r=d["roofline"]
    print(v, cl, round(d["ms_per_step"],1), round(r["loop_ms"],1), round(r["frac"],4))
except Exception as e: print(v, cl, "failed", open(f"gpurun_out/c5_{v}_{cl}.log").read()[-300:])
PY
  done
done
cp /tmp/keep.so paper_2203_02507_b200/lib/libfpm_b200.so
