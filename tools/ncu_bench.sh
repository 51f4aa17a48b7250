#!/bin/bash
# ncu evidence for the bench workload (run on the GPU box after bench.py itself exited 0):
#  1) launch list of one step (gpu__time_duration per kernel, serialised, cold-ish)
#  2) --set full of the loop kernel with source-line attribution
# usage: tools/ncu_bench.sh <tag> [bench args]
tag=$1; shift
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 "$@" > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fpm_loop -s 3 -c 1 \
  -o gpurun_out/ncu_loop_$tag python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 "$@" > gpurun_out/ncu_full_$tag.log 2>&1
echo "$tag done"
