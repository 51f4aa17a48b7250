python tools/quad_check.py > gpurun_out/quad_check.txt 2>&1
for v in "QUAD=0" "QUAD=1 QMINB=2"; do
  env $(echo $v | sed 's/\([A-Z]*=\)/FPM_B200_\1/g') python tools/strong_probe.py --gpus 1 2 4 8 > gpurun_out/probe_tmp.txt 2>&1
  echo "== $v" >> gpurun_out/quad_probe.txt; cat gpurun_out/probe_tmp.txt >> gpurun_out/quad_probe.txt
done
cat gpurun_out/quad_check.txt gpurun_out/quad_probe.txt
