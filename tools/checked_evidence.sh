#!/bin/bash
# On the GPU box: the bounds-checked build's evidence for profiles/ (compute-sanitizer
# substitute): every path clean under the asserts, the race-jitter suite on the
# checked build, and the self-test trap.
out=gpurun_out/checked_build.txt
: > $out
echo "== tests/checked_cases.py under FPM_B200_LIB=check" >> $out
FPM_B200_LIB=check timeout 900 python tests/checked_cases.py /tmp/checked.npz >> $out 2>&1; echo "exit $?" >> $out
echo "== tests/test_race_jitter.py under FPM_B200_LIB=check (jitter + bounds asserts)" >> $out
FPM_B200_LIB=check timeout 1200 python -m pytest tests/test_race_jitter.py -q -m gpu >> $out 2>&1; echo "exit $?" >> $out
echo "== self-test (FPM_B200_CHECK_SELFTEST=1: tile count 0, the tile assert must trap)" >> $out
FPM_B200_LIB=check FPM_B200_CHECK_SELFTEST=1 timeout 300 python -c "
import paper_2203_02507_b200 as fpm
from tests.helpers import dataset, gpu_cfg
cfg = gpu_cfg(led_scan_rows=3, led_scan_cols=3)
fs, _, seq, _ = dataset(cfg, seed=80)
t = fpm.partition_tiles(64, 64, cfg)[0]
fpm.reconstruct_tile(fs, t, cfg, 1, seq, engine=fpm.Engine(0))
print('NO TRAP')" >> $out 2>&1; echo "exit $? (non-zero expected)" >> $out
