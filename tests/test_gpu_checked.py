"""Bounds-checked build (the memcheck half of compute-sanitizer, which this GPU
pool does not allow: profiles/r2/compute_sanitizer_refused.txt).

libfpm_b200_check.so (make check, -DFPM_CHECK=1) asserts on the device the
tile, origin (the n x n disk block inside the N x N canvas), frame, work-item,
slab-row / slab-owner and measurement-slot index of every kernel's global and
shared accesses, and traps on a violation. tests/checked_cases.py runs every
kernel family and host path under it in a subprocess (a trap would surface as a
CUDA error and a non-zero exit); its results must equal the production
build's. The disjoint-disk contract behind the races is recon.cpp:105-106."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_2203_02507_b200", "lib", "libfpm_b200_check.so")

pytestmark = pytest.mark.gpu


def test_checked_build_runs_every_path_clean(tmp_path):
    assert os.path.exists(CHECK_LIB), "run __graft_entry__.build() (make check)"
    out = tmp_path / "checked.npz"
    env = dict(os.environ, FPM_B200_LIB="check")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_cases.py"), str(out)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-4000:])
    assert "FPM_ASSERT" not in p.stdout + p.stderr
    assert "libfpm_b200_check.so" in p.stdout
    got = np.load(out)

    from tests import checked_cases
    ref = checked_cases.run_all()
    assert sorted(ref) == sorted(got.files)
    for k, v in ref.items():
        g = got[k]
        assert g.shape == v.shape, k
        scale = float(np.abs(v).max()) or 1.0
        # the asserts add instructions, not arithmetic: the same values (tolerance only
        # for a compiler contracting differently around them)
        assert float(np.abs(g - v).max()) <= 1e-5 * scale, k


def test_checked_build_traps_on_a_bad_index():
    """The asserts are live: FPM_B200_CHECK_SELFTEST=1 hands the loop kernel a tile
    count of 0 (checked build only), so its tile assert must trap and the call
    must fail loudly instead of returning results."""
    code = ("import numpy as np, paper_2203_02507_b200 as fpm\n"
            "from tests.helpers import dataset, gpu_cfg\n"
            "cfg = gpu_cfg(led_scan_rows=3, led_scan_cols=3)\n"
            "fs, _, seq, _ = dataset(cfg, seed=80)\n"
            "t = fpm.partition_tiles(64, 64, cfg)[0]\n"
            "fpm.reconstruct_tile(fs, t, cfg, 1, seq, engine=fpm.Engine(0))\n"
            "print('NO TRAP')\n")
    env = dict(os.environ, FPM_B200_LIB="check", FPM_B200_CHECK_SELFTEST="1")
    p = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode != 0 and "NO TRAP" not in p.stdout, (p.stdout[-1000:], p.stderr[-2000:])
