#!/bin/bash
# On the GPU box: tools/strong_probe.py (config 3, 8/2/1 GPUs' worth of tiles) for every
# lib_v/<variant>/libfpm_b200.so, appended to gpurun_out/probe_v.txt; restores the
# in-tree library afterwards.
cp paper_2203_02507_b200/lib/libfpm_b200.so /tmp/keep.so
for d in lib_v/*/; do
  v=$(basename "$d")
  cp "$d/libfpm_b200.so" paper_2203_02507_b200/lib/libfpm_b200.so
  echo "== $v" >> gpurun_out/probe_v.txt
  timeout 300 python tools/strong_probe.py --config 3 --gpus 8 2 1 >> gpurun_out/probe_v.txt 2>&1
done
cp /tmp/keep.so paper_2203_02507_b200/lib/libfpm_b200.so
