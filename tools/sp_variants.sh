cp paper_2203_02507_b200/lib/libfpm_b200.so /tmp/keep.so
for v in base q1; do
  if [ $v != base ]; then cp lib_v/$v/libfpm_b200.so paper_2203_02507_b200/lib/libfpm_b200.so; fi
  echo "== $v" >> gpurun_out/sp_variants.txt
  python tools/strong_probe.py --gpus 4 8 >> gpurun_out/sp_variants.txt 2>&1
  cp /tmp/keep.so paper_2203_02507_b200/lib/libfpm_b200.so
done
