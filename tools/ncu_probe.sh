#!/bin/bash
# ncu --set full of the n = 64 loop kernel on one strong-scaled rank's band (config 3, G ranks)
# usage: tools/ncu_probe.sh <tag> <G> [env assignments...]
tag=$1; G=$2; shift 2
env "$@" timeout 900 ncu --set full --import-source on --clock-control none -k regex:fpm_loop64 -s 1 -c 1 \
  -o gpurun_out/ncu_$tag python tools/strong_probe.py --gpus $G --steps 1 > gpurun_out/ncu_$tag.log 2>&1
echo "$tag rc=$?" >> gpurun_out/ncu_summary.txt
