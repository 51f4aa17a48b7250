"""Committed golden fixtures (tests/golden/, made by make_golden.py from the
oracle): the oracle must keep reproducing them (CPU), and the device path must
match them (GPU) — parity that does not depend on rebuilding the oracle."""
import json
import os

import numpy as np
import pytest

import paper_2203_02507_b200 as fpm
from tests.helpers import amp_phase_rel

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["toy3x3_gs", "c1_7x7_gs", "epry_9x9_defocus25", "n128_7x7_epry"]


def _load(name):
    return dict(np.load(os.path.join(HERE, f"{name}.npz")))


def _cfg(name):
    from tests.golden.make_golden import CASES as C
    tile, ov, scan, fov, seed, dz, order, iters, mode, stride = C[name]
    return fpm.OpticalConfig(tile_size=tile, tile_overlap=ov, upsample=4, led_scan_rows=scan,
                             led_scan_cols=scan), iters, mode


def test_reference_literals_fixture(orc):
    lit = json.load(open(os.path.join(HERE, "reference_literals.json")))
    for key, d in lit.items():
        if "rel" in d:
            assert d["value"] == pytest.approx(d["expect"], rel=d["rel"]), key
        else:
            assert d["value"] == d["expect"], key


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_fixture(orc, name):
    from tests.golden.make_golden import case
    g = _load(name)
    cfg, fs, seq, r, stride = case(name)
    assert np.array_equal(fs.images, g["frames"])
    assert np.array_equal(np.asarray(seq, np.int32), g["seq"])
    assert np.abs(r.hr[::stride, ::stride] - g["hr"]).max() <= 1e-6 * np.abs(g["hr"]).max()
    assert np.allclose(r.residuals, g["residuals"], rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_matches_fixture(name):
    g = _load(name)
    cfg, iters, mode = _cfg(name)
    fs = fpm.FrameSet(g["frames"], [tuple(x) for x in g["leds"].tolist()])
    seq = [tuple(x) for x in g["seq"].tolist()]
    t = fpm.partition_tiles(fs.width(), fs.height(), cfg)[0]
    got = fpm.reconstruct_tile(fs, t, cfg, iters, seq, mode=mode)
    s = int(g["hr_stride"])
    amp, ph = amp_phase_rel(got.hr[::s, ::s], g["hr"])
    assert amp < 1e-4 and ph < 1e-4, (amp, ph)
    assert np.allclose(got.metrics.pass_mean_residual, g["residuals"], rtol=1e-3)
    if mode == "epry":
        assert np.linalg.norm(got.pupil - g["pupil"]) / np.linalg.norm(g["pupil"]) < 1e-4


@pytest.mark.gpu
def test_device_mosaic_matches_fixture():
    g = _load("mosaic120_5x5_gs")
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=8, upsample=4, led_scan_rows=5, led_scan_cols=5)
    fs = fpm.FrameSet(g["frames"], [tuple(x) for x in g["leds"].tolist()])
    seq = [tuple(x) for x in g["seq"].tolist()]
    res = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=2))
    amp, ph = amp_phase_rel(res.stitched[::2, ::2], g["stitched"])
    assert amp < 1e-4 and ph < 1e-4, (amp, ph)
    assert np.allclose(np.array([m.pass_mean_residual for m in res.tile_metrics]), g["residuals"], rtol=1e-3)
