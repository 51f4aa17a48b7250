cd $GRAFT_REPO_ROOT
./tools/pipe_rates > gpurun_out/pipe_rates.txt 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for spec in "racecheck loop64_queue" "racecheck loop64" "synccheck loop64_queue" "synccheck cluster128" "racecheck cluster128" "synccheck cluster256" "memcheck host_banded" "memcheck mosaic" "memcheck loop64_queue" "memcheck cluster256"; do
  set -- $spec
  timeout 900 $CS --tool $1 --print-limit 20 python tools/sanitize_case.py $2 > gpurun_out/san_$1_$2.log 2>&1
  echo "$1 $2 rc=$?" >> gpurun_out/san_summary.txt
done
cat gpurun_out/pipe_rates.txt gpurun_out/san_summary.txt
