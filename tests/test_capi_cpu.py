"""CPU-side checks of libfpm_b200.so: it loads, exports every symbol the header
declares, and its host geometry (the integers the kernels consume) is
bit-exact against the oracle and the reference literals. No device calls."""
import os
import re

import numpy as np
import pytest

import paper_2203_02507_b200 as fpm
from paper_2203_02507_b200 import _lib
from tests.helpers import orc_cfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "fpm_b200.h")).read()
    declared = set(re.findall(r"\b(fpmgpu_[a-z_0-9]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    L = _lib.lib()
    for name in sorted(declared):
        assert hasattr(L, name), f"{name} declared in fpm_b200.h but not exported"
    assert set(_lib.EXPORTS) == declared
    assert L.fpmgpu_version() >= 1


def test_default_config_matches_reference():
    import ctypes
    c = _lib.OpticalConfigC()
    _lib.lib().fpmgpu_default_config(ctypes.byref(c))
    d = fpm.OpticalConfig()
    for f, _ in _lib.OpticalConfigC._fields_:
        assert getattr(c, f) == pytest.approx(getattr(d, f)), f


def test_reference_literals():
    c = fpm.OpticalConfig()
    fx, fy = fpm.illumination_wavevector((32, 33), (0, 0), c)
    assert fx == pytest.approx(-0.0573463, rel=1e-5) and fy == 0.0
    assert fpm.spectrum_offset_px((fx, fy), c) == (0, -18)  # test_forward.cpp:92-98
    assert fpm.build_pupil(c, 256).radius_px == pytest.approx(58.514, rel=1e-4)  # test_optics.cpp:83
    assert fpm.synthesized_na(c) == pytest.approx(0.34762, rel=1e-4)  # test_optics.cpp:121
    assert fpm.tile_origins(2048, 256, 26) == [0, 230, 460, 690, 920, 1150, 1380, 1610, 1792]
    assert fpm.sequence_offsets("spiral", 3, 3) == [(0, 0), (0, 1), (-1, 1), (-1, 0), (-1, -1), (0, -1),
                                                    (1, -1), (1, 0), (1, 1)]
    toy = fpm.OpticalConfig(tile_size=64, tile_overlap=8, led_scan_rows=3, led_scan_cols=3)
    t = fpm.partition_tiles(64, 64, toy)[0]
    assert fpm.min_safe_lag_tile(fpm.led_sequence("spiral", toy), t, toy) == 9  # test_parallel.cpp:61
    assert fpm.min_safe_lag([(0, 0)] * 5, 3.0) == 5
    grid = [(10 * r, 10 * cc) for r in (-1, 0, 1) for cc in (-1, 0, 1)]
    assert fpm.min_safe_lag(grid, 7.0) == 4


def test_errors_carry_reference_messages():
    with pytest.raises(fpm.ConfigError, match="pupil exceeds Nyquist"):
        fpm.build_pupil(fpm.OpticalConfig(objective_na=0.9), 64)
    with pytest.raises(fpm.DomainError):
        fpm.illumination_wavevector((64, 0), (0, 0), fpm.OpticalConfig())
    with pytest.raises(fpm.ConfigError):
        fpm.OpticalConfig(upsample=1).validate()
    with pytest.raises(fpm.ConfigError):
        fpm.tile_origins(100, 256, 26)
    with pytest.raises(fpm.ConfigError):
        fpm.sequence_offsets("spiral", 4, 3)


@pytest.mark.parametrize("fov,tile,ov,scan", [(2048, 64, 0, 15), (4096, 256, 0, 21), (2048, 256, 26, 13),
                                              (170, 64, 8, 3)])
def test_offsets_bit_exact_vs_oracle(orc, fov, tile, ov, scan):
    """North-star check 1: LED-to-spectrum offsets and sub-aperture origins bit-exact."""
    cfg = fpm.OpticalConfig(tile_size=tile, tile_overlap=ov, led_scan_rows=scan, led_scan_cols=scan,
                            center_row=32, center_col=32)
    seq = fpm.led_sequence("spiral", cfg)
    assert seq == orc.led_sequence("spiral", orc_cfg(cfg))
    xy, ce, kv, of = fpm.partition_arrays(fov, fov, cfg, seq)
    ref = orc.partition_tiles(fov, fov, orc_cfg(cfg), seq)
    assert np.array_equal(xy, ref.xy)
    assert np.array_equal(ce, ref.center)
    assert np.array_equal(kv, ref.kvecs)
    assert np.array_equal(of, ref.offsets)


def test_pupil_and_schedule_vs_oracle(orc):
    cfg = fpm.OpticalConfig()
    for grid, z in ((64, 0.0), (64, 30.0), (128, -12.5), (256, 0.0)):
        p = fpm.build_pupil(cfg, grid, z)
        v, r = orc.build_pupil(orc_cfg(cfg), grid, z)
        assert p.radius_px == r
        assert np.array_equal(p.values != 0, v != 0)
        assert np.abs(p.values - v).max() < 1e-15
    for lag in (1, 2, 5, 9):
        s = fpm.build_schedule(9, 3, lag)
        rounds, ent = orc.build_schedule(9, 3, lag)
        assert len(s.rounds) == rounds
        got = sorted((r, st, p) for r, rr in enumerate(s.rounds) for st, p in rr)
        assert got == sorted(map(tuple, ent.tolist()))


def test_missing_frame_is_data_error():
    cfg = fpm.OpticalConfig(tile_size=64, led_scan_rows=3, led_scan_cols=3)
    fs = fpm.FrameSet(np.zeros((1, 64, 64), np.uint16), [cfg.center_led])
    t = fpm.partition_tiles(64, 64, cfg)
    with pytest.raises(fpm.DataError, match="missing frame"):
        fpm.make_request(fs, cfg, fpm.led_sequence("spiral", cfg), t, 1)


def test_stitch_mosaic_size_query():
    """Mosaic extents from the device stitch's host layout (no device work):
    4x4 stock tiles span 946 px (test_stitch.cpp:148-161), toy FOV 120 -> 480."""
    import ctypes
    L = _lib.lib()
    for cfg, fov in ((fpm.OpticalConfig(upsample=1), 946), (fpm.OpticalConfig(tile_size=64, tile_overlap=8), 120)):
        specs = fpm.partition_tiles(fov, fov, cfg)
        xy = np.ascontiguousarray([[s.x0, s.y0] for s in specs], np.int32)
        r, c = ctypes.c_int(), ctypes.c_int()
        cc = cfg.c()
        _lib.check(L.fpmgpu_stitch_mosaic(None, ctypes.byref(cc), None, xy.ctypes.data, len(xy), None,
                                          ctypes.byref(r), ctypes.byref(c)))
        assert (r.value, c.value) == (fov * cfg.upsample, fov * cfg.upsample)
