"""Pins the CPU oracle against the reference's own known-answer tests.

Each test names the reference test it re-expresses (proj/tests/*.cpp:line).
The reference cannot be built here (no Eigen), so these literals and
properties are what anchors the oracle, and through it every GPU parity test.
"""
import math

import numpy as np
import pytest

from oracle.oracle import (ConfigError, DataError, DomainError, Optics, UnsafeLagError, toy_cfg)


def rand_field(rows, cols, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (rows, cols)) + 1j * rng.uniform(-1, 1, (rows, cols))


# ---------------------------------------------------------------- test_field.cpp
def test_dc_term_centered(orc):  # test_field.cpp:26-36
    spec = orc.fft2(np.ones((8, 8), complex))
    assert abs(spec[4, 4] - 64) < 1e-12
    spec[4, 4] = 0
    assert np.abs(spec).max() < 1e-9


def test_round_trip(orc):  # test_field.cpp:38-42
    x = rand_field(64, 64, 7)
    assert np.abs(orc.ifft2(orc.fft2(x)) - x).max() / np.abs(x).max() < 1e-12


def test_parseval(orc):  # test_field.cpp:44-51
    x = rand_field(32, 32, 11)
    X = orc.fft2(x)
    assert np.sum(np.abs(X) ** 2) == pytest.approx(np.sum(np.abs(x) ** 2) * 32 * 32, rel=1e-12)


def test_linearity(orc):  # test_field.cpp:53-59
    x, y = rand_field(16, 16, 1), rand_field(16, 16, 2)
    a = 0.7 - 1.3j
    lhs = orc.fft2(a * x + y)
    rhs = a * orc.fft2(x) + orc.fft2(y)
    assert np.abs(lhs - rhs).max() / np.abs(rhs).max() < 1e-12


def test_threaded_bit_exact(orc):  # test_field.cpp:61-65
    x = rand_field(64, 64, 3)
    assert np.array_equal(orc.fft2(x, 1), orc.fft2(x, 4))
    assert np.array_equal(orc.ifft2(x, 1), orc.ifft2(x, 3))


def test_shift_positions(orc):  # test_field.cpp:67-73
    x = rand_field(9, 9, 5)
    assert np.array_equal(orc.fftshift(orc.fftshift(x), inverse=True), x)
    d = np.zeros((8, 8), complex)
    d[0, 0] = 1
    assert orc.fftshift(d)[4, 4] == 1


def test_bilinear_constant(orc):  # test_field.cpp:75-80
    up = orc.upsample_bilinear(np.full((16, 16), 3.5), 4)
    assert up.shape == (64, 64)
    assert np.abs(up - 3.5).max() < 1e-12


@pytest.mark.parametrize("n", [6, 10, 12, 15, 30, 48, 96, 384, 480, 7 * 11, 13 * 4])
def test_mixed_radix_matches_numpy(orc, n):
    # simulate_dataset needs non-power-of-two sizes (forward.cpp:218-221)
    x = rand_field(n, n, n)
    ref = np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x)))
    assert np.abs(orc.fft2(x) - ref).max() / np.abs(ref).max() < 1e-12
    ref_i = np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(x)))
    assert np.abs(orc.ifft2(x) - ref_i).max() / np.abs(ref_i).max() < 1e-12


# ---------------------------------------------------------------- test_optics.cpp
def test_config_invariants(orc):  # test_optics.cpp:15-30
    orc.validate(Optics())
    for bad in (dict(tile_overlap=256), dict(upsample=1), dict(led_scan_rows=12),
                dict(center_row=1, center_col=1)):
        with pytest.raises(ConfigError):
            orc.validate(Optics(**bad))
    assert Optics().dx_obj == pytest.approx(1.2)


def test_on_axis_zero(orc):  # test_optics.cpp:32-36
    assert orc.illumination_wavevector((32, 32), (0, 0), Optics()) == (0.0, 0.0)


def test_one_pitch_fx(orc):  # test_optics.cpp:38-46
    c = Optics()
    fx, fy = orc.illumination_wavevector((32, 33), (0, 0), c)
    sin_t = 2.5 / math.sqrt(2.5 ** 2 + 83.0 ** 2)
    assert fx == pytest.approx(-sin_t / c.wavelength, rel=1e-12)
    assert fx == pytest.approx(-0.0573463, rel=1e-5)
    assert fy == 0.0


def test_edge_led_sin(orc):  # test_optics.cpp:48-52
    c = Optics()
    fx, _ = orc.illumination_wavevector((32, 38), (0, 0), c)
    assert c.wavelength * abs(fx) == pytest.approx(0.177842, rel=1e-5)


def test_led_domain_error(orc):  # test_optics.cpp:54-57
    with pytest.raises(DomainError):
        orc.illumination_wavevector((64, 0), (0, 0), Optics())
    with pytest.raises(DomainError):
        orc.illumination_wavevector((0, -1), (0, 0), Optics())


def test_evanescent_exclusion(orc):  # test_optics.cpp:59-69
    c = Optics()
    lim = 1.0 / c.wavelength ** 2
    for dr in range(-6, 7):
        for dc in range(-6, 7):
            for cx in (-1000.0, 0.0, 1000.0):
                fx, fy = orc.illumination_wavevector((32 + dr, 32 + dc), (cx, -cx), c)
                assert fx * fx + fy * fy < lim


def test_distinct_tile_centers(orc):  # test_optics.cpp:71-77
    c = Optics()
    a = orc.illumination_wavevector((34, 31), (0, 0), c)
    b = orc.illumination_wavevector((34, 31), (300.0, 0), c)
    assert a[0] != b[0]


def test_pupil_radius_and_support(orc):  # test_optics.cpp:79-101
    vals, radius = orc.build_pupil(Optics(), 256, 0.0)
    assert radius == pytest.approx(58.514, rel=1e-4)
    i, j = np.mgrid[0:256, 0:256]
    inside = np.hypot(i - 128.0, j - 128.0) <= radius
    assert np.all(vals[inside] == 1) and np.all(vals[~inside] == 0)
    assert abs(inside.sum() - math.pi * radius ** 2) < 2 * math.pi * radius


def test_pupil_conjugate_defocus(orc):  # test_optics.cpp:103-109
    a, _ = orc.build_pupil(Optics(), 64, 30.0)
    b, _ = orc.build_pupil(Optics(), 64, -30.0)
    assert np.abs(a - b.conj()).max() < 1e-15
    assert np.all(np.abs(a) <= 1 + 1e-15)


def test_pupil_nyquist_refusal(orc):  # test_optics.cpp:111-117
    with pytest.raises(ConfigError, match="pupil exceeds Nyquist"):
        orc.build_pupil(Optics(objective_na=0.9), 64, 0.0)
    with pytest.raises(ConfigError):
        orc.build_pupil(Optics(), 31, 0.0)


def test_synthesized_na(orc):  # test_optics.cpp:119-124
    assert orc.synthesized_na(Optics()) == pytest.approx(0.34762, rel=1e-4)
    assert orc.synthesized_na(Optics(led_scan_rows=1, led_scan_cols=1)) == pytest.approx(0.1)


# ---------------------------------------------------------------- test_recon.cpp orders
def test_raster_3x3(orc):  # test_recon.cpp:13-20
    s = orc.sequence_offsets("raster", 3, 3)
    assert len(s) == 9 and s[0] == (-1, -1) and s[1] == (-1, 0) and s[4] == (0, 0) and s[8] == (1, 1)


def test_spiral_3x3(orc):  # test_recon.cpp:22-27
    assert orc.sequence_offsets("spiral", 3, 3) == [
        (0, 0), (0, 1), (-1, 1), (-1, 0), (-1, -1), (0, -1), (1, -1), (1, 0), (1, 1)]


def test_spiral_rectangular(orc):  # test_recon.cpp:29-38
    s = orc.sequence_offsets("spiral", 5, 3)
    assert len(s) == 15 and len(set(s)) == 15
    assert all(abs(r) <= 2 and abs(c) <= 1 for r, c in s)


def test_spiral_1x1_even_refused(orc):  # test_recon.cpp:40-45
    assert orc.sequence_offsets("spiral", 1, 1) == [(0, 0)]
    with pytest.raises(ConfigError):
        orc.sequence_offsets("spiral", 4, 3)


# ---------------------------------------------------------------- test_forward.cpp
def test_one_pitch_offset_minus_18(orc):  # test_forward.cpp:92-98
    c = Optics()
    kv = orc.illumination_wavevector((32, 33), (0, 0), c)
    assert orc.spectrum_offset_px(kv, c) == (0, -18)


def test_phase_disk_object(orc):  # test_forward.cpp:13-19
    obj = orc.synth_object("phase-disk", 256, 0)
    assert np.abs(np.abs(obj) - 1).max() < 1e-15
    assert np.angle(obj[128, 128]) == pytest.approx(math.pi / 2)
    assert np.angle(obj[128, 168]) == pytest.approx(0.0)
    assert np.angle(obj[128, 148]) == pytest.approx(math.pi / 2)


def test_objects_deterministic_and_bounded(orc):  # test_forward.cpp:36-58
    for k in ("bars", "phase-disk", "composite"):
        assert np.array_equal(orc.synth_object(k, 256, 42), orc.synth_object(k, 256, 42))
    assert not np.array_equal(orc.synth_object("composite", 256, 1), orc.synth_object("composite", 256, 2))
    obj = orc.synth_object("composite", 256, 9)
    assert np.abs(obj).min() >= 0.1 and np.abs(obj).max() <= 1.0
    assert np.abs(np.angle(obj)).max() <= math.pi / 2


def test_flat_frame_constant(orc):  # test_forward.cpp:60-69 (via simulate_dataset)
    cfg = toy_cfg()
    flat = np.ones((cfg.hr_size, cfg.hr_size), complex)
    fs = orc.simulate_dataset(flat, [cfg.center_led], cfg)
    img = fs.images[0].astype(int)
    assert img[0, 0] == pytest.approx(0.8 * 65535, rel=0.01)
    assert np.abs(img - img[0, 0]).max() <= 1


def test_offset_equals_pretilt(orc):  # test_forward.cpp:71-90
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 3)
    dk = 1.0 / (cfg.tile_size * cfg.dx_obj)
    kv = (3 * dk, -2 * dk)
    via_offset = orc.simulate_intensity(obj, kv, cfg)
    n = cfg.hr_size
    dx = cfg.dx_obj / cfg.upsample
    i, j = np.mgrid[0:n, 0:n]
    x, y = (j - n // 2) * dx, (i - n // 2) * dx
    tilted = obj * np.exp(-2j * math.pi * (kv[0] * x + kv[1] * y))
    via_tilt = orc.simulate_intensity(tilted, (0, 0), cfg)
    assert np.abs(via_offset - via_tilt).max() / via_offset.max() < 1e-10


def test_headroom_refusal(orc):  # test_forward.cpp:100-107
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 3)
    with pytest.raises(DataError, match="illumination NA too high"):
        orc.simulate_intensity(obj, (0.95 / cfg.wavelength, 0), cfg)


def test_flat_9_equal_frames(orc):  # test_forward.cpp:109-117
    cfg = toy_cfg()
    flat = np.ones((cfg.hr_size, cfg.hr_size), complex)
    fs = orc.simulate_dataset(flat, orc.led_sequence("raster", cfg), cfg)
    assert len(fs.leds) == 9
    for f in fs.images:
        assert np.abs(f.astype(int) - fs.images[0].astype(int)).max() <= 1


def test_timestamps(orc):  # test_forward.cpp:119-128
    cfg = toy_cfg()
    fs = orc.simulate_dataset(orc.synth_object("composite", cfg.hr_size, 5), orc.led_sequence("spiral", cfg), cfg)
    step = cfg.acq_pattern_delay + cfg.acq_exposure
    assert np.allclose(fs.timestamps, (np.arange(9) + 1) * step)
    assert 169 * step == pytest.approx(55.77)


def test_noise_determinism(orc):  # test_forward.cpp:154-172
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 11)
    seq = orc.led_sequence("spiral", cfg)
    a = orc.simulate_dataset(obj, seq, cfg)
    b = orc.simulate_dataset(obj, seq, cfg)
    assert np.array_equal(a.images, b.images)
    c = orc.simulate_dataset(obj, seq, cfg, noise=(1e4, 77))
    d = orc.simulate_dataset(obj, seq, cfg, noise=(1e4, 77))
    assert np.array_equal(c.images, d.images) and not np.array_equal(c.images, a.images)


def test_on_axis_lowpass_decimate(orc):  # test_forward.cpp:174-192
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 13)
    _, radius = orc.build_pupil(cfg, cfg.tile_size, 0.0)
    sim = orc.simulate_intensity(obj, (0, 0), cfg)
    N, up = cfg.hr_size, cfg.upsample
    spec = orc.fft2(obj)
    i, j = np.mgrid[0:N, 0:N]
    spec[np.hypot(i - N / 2, j - N / 2) > radius] = 0
    filt = orc.ifft2(spec)
    ref = np.abs(filt[::up, ::up]) ** 2
    assert np.abs(sim / sim.max() - ref / ref.max()).max() < 1e-9


# ---------------------------------------------------------------- test_recon.cpp
def test_flat_init_dc_only(orc):  # test_recon.cpp:56-66
    cfg = toy_cfg()
    flat = np.ones((cfg.hr_size, cfg.hr_size), complex)
    fs = orc.simulate_dataset(flat, [cfg.center_led], cfg)
    canvas = orc.init_canvas(fs, cfg)
    c = canvas.shape[0] // 2
    dc = abs(canvas[c, c])
    canvas[c, c] = 0
    assert dc > 0 and np.abs(canvas).max() / dc < 1e-10


def test_zero_iter_round_trip(orc):  # test_recon.cpp:77-86
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 2)
    fs = orc.simulate_dataset(obj, [cfg.center_led], cfg)
    canvas = orc.init_canvas(fs, cfg)
    expected = orc.upsample_bilinear(np.sqrt(fs.images[0].astype(float)), cfg.upsample)
    out = orc.canvas_to_field(canvas, cfg)
    assert np.abs(np.abs(out) - expected).max() / expected.max() < 1e-12


def test_brightest_fallback(orc):  # test_recon.cpp:88-94
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 2)
    fs = orc.simulate_dataset(obj, [(32, 33)], cfg)
    orc.init_canvas(fs, cfg)




def test_fixed_point(orc):  # test_recon.cpp:96-116
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 3)
    fs = orc.simulate_dataset(obj, [cfg.center_led], cfg)
    canvas = orc.init_canvas(fs, cfg)
    pupil, _ = orc.build_pupil(cfg, cfg.tile_size, 0.0)
    tiles = orc.partition_tiles(cfg.tile_size, cfg.tile_size, cfg, [(32, 33)])
    kv = tuple(tiles.kvecs[0, 0])
    oy, ox = orc.spectrum_offset_px(kv, cfg)
    n, N = cfg.tile_size, cfg.hr_size
    r0, c0 = N // 2 + oy - n // 2, N // 2 + ox - n // 2
    block = canvas[r0:r0 + n, c0:c0 + n] * pupil
    intensity = np.abs(orc.ifft2(block)) ** 2
    before = canvas.copy()
    res = orc.update_step(canvas, intensity, kv, pupil, cfg)
    assert res <= 1e-12
    assert np.abs(before - canvas).max() / np.abs(before).max() <= 1e-10


def test_support_confinement(orc):  # test_recon.cpp:118-145
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 4)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    canvas = orc.init_canvas(fs, cfg)
    init = canvas.copy()
    pupil, radius = orc.build_pupil(cfg, cfg.tile_size, 0.0)
    tiles = orc.partition_tiles(fs.width, fs.height, cfg, seq)
    n, N = cfg.tile_size, cfg.hr_size
    for k, led in enumerate(seq):
        I = fs.images[fs.find(led)][0:n, 0:n].astype(float)
        orc.update_step(canvas, I, tuple(tiles.kvecs[0, k]), pupil, cfg)
    i, j = np.mgrid[0:N, 0:N]
    inside = np.zeros((N, N), bool)
    for oy, ox in tiles.offsets[0]:
        inside |= np.hypot(i - (N // 2 + oy), j - (N // 2 + ox)) <= radius
    assert np.array_equal(canvas[~inside], init[~inside])  # bit-exact


def test_pass2_not_worse(orc):  # test_recon.cpp:147-155
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 5)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    r = orc.reconstruct_tile(fs, cfg, 2, seq)
    assert r.residuals[1] <= r.residuals[0]


def test_degenerate_aperture(orc):  # test_recon.cpp:157-167
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 6)
    fs = orc.simulate_dataset(obj, [cfg.center_led], cfg)
    r = orc.reconstruct_tile(fs, cfg, 1, [cfg.center_led])
    expected = orc.upsample_bilinear(np.sqrt(fs.images[0].astype(float)), cfg.upsample)
    rel = np.sqrt(np.mean((np.abs(r.hr) - expected) ** 2)) / expected.max()
    assert rel < 0.03


def test_toy_9x9_recovers(orc):  # test_recon.cpp:169-181
    cfg = toy_cfg(led_scan_rows=9, led_scan_cols=9)
    obj = orc.synth_object("composite", cfg.hr_size, 8)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    r = orc.reconstruct_tile(fs, cfg, 5, seq)
    truth = orc.band_limit(obj, orc.synthesized_na(cfg), cfg)
    aligned = r.hr * orc.global_alignment(r.hr, truth)
    amp, ph = orc.rmse(aligned, truth)
    assert amp <= 0.03 and ph <= 0.1


def test_missing_frame(orc):  # test_recon.cpp:183-190
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 6)
    fs = orc.simulate_dataset(obj, [cfg.center_led], cfg)
    with pytest.raises(DataError, match="missing frame"):
        orc.reconstruct_tile(fs, cfg, 1, orc.led_sequence("spiral", cfg))


# ---------------------------------------------------------------- test_parallel.cpp
def test_lag_literals(orc):  # test_parallel.cpp:14-32
    assert orc.min_safe_lag([(0, 0)] * 5, 3.0) == 5
    assert orc.min_safe_lag([(0, 0), (0, 100), (0, 200), (0, 300)], 10.0) == 1
    grid = [(10 * r, 10 * c) for r in (-1, 0, 1) for c in (-1, 0, 1)]
    assert orc.min_safe_lag(grid, 7.0) == 4


def test_lag_brute_force(orc):  # test_parallel.cpp:34-54
    rng = np.random.default_rng(2024)
    for trial in range(50):
        offs = [tuple(x) for x in rng.integers(-40, 41, (12, 2)).tolist()]
        radius = 5.0 + trial % 7
        gap = 0
        for i in range(12):
            for j in range(i, 12):
                if math.hypot(offs[i][0] - offs[j][0], offs[i][1] - offs[j][1]) < 2 * radius:
                    gap = max(gap, j - i)
        assert orc.min_safe_lag(offs, radius) == 1 + gap


def test_toy_lag_9(orc):  # test_parallel.cpp:56-62
    cfg = toy_cfg()
    assert orc.min_safe_lag_tile(cfg, 64, 64, 0, orc.led_sequence("spiral", cfg)) == 9


def test_schedule_coverage(orc):  # test_parallel.cpp:64-77
    for lag in (1, 2, 5, 9):
        rounds, ent = orc.build_schedule(9, 3, lag)
        assert rounds == 9 + 2 * lag
        assert np.all(ent[:, 2] + ent[:, 1] * lag == ent[:, 0])
        assert len({(s, p) for _, s, p in ent.tolist()}) == 27


def test_pipelined_lag_ge_L_identical(orc):  # test_parallel.cpp:79-95
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 21)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    a = orc.reconstruct_tile(fs, cfg, 3, seq)
    b = orc.reconstruct_tile(fs, cfg, 3, seq, pipelined=True, lag=len(seq))
    assert np.array_equal(a.hr, b.hr)
    assert np.allclose(a.residuals, b.residuals, rtol=1e-12, atol=0)


def test_pipelined_auto_identical(orc):  # test_parallel.cpp:97-108
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 22)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    a = orc.reconstruct_tile(fs, cfg, 3, seq)
    b = orc.reconstruct_tile(fs, cfg, 3, seq, pipelined=True)
    assert b.lag == orc.min_safe_lag_tile(cfg, 64, 64, 0, seq) and not b.nondeterministic
    assert np.array_equal(a.hr, b.hr)


def test_pipelined_wide_scan_identical(orc):  # test_parallel.cpp:110-122
    cfg = toy_cfg(led_scan_rows=7, led_scan_cols=7)
    obj = orc.synth_object("composite", cfg.hr_size, 23)
    seq = orc.led_sequence("raster", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    lag = orc.min_safe_lag_tile(cfg, 64, 64, 0, seq)
    assert lag < len(seq)
    a = orc.reconstruct_tile(fs, cfg, 2, seq)
    b = orc.reconstruct_tile(fs, cfg, 2, seq, pipelined=True, lag=lag)
    assert np.array_equal(a.hr, b.hr)


def test_unsafe_lag(orc):  # test_parallel.cpp:124-141
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 24)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    with pytest.raises(UnsafeLagError) as ei:
        orc.reconstruct_tile(fs, cfg, 2, seq, pipelined=True, lag=1)
    assert ei.value.minimum == 9
    f = orc.reconstruct_tile(fs, cfg, 2, seq, pipelined=True, lag=1, force_unsafe=True)
    assert f.nondeterministic and f.lag == 1 and np.all(np.isfinite(f.hr))


def test_tile_origins_literals(orc):  # test_parallel.cpp:143-149
    assert orc.tile_origins(2048, 256, 26) == [0, 230, 460, 690, 920, 1150, 1380, 1610, 1792]
    assert orc.tile_origins(256, 256, 26) == [0]
    assert orc.tile_origins(486, 256, 26) == [0, 230]
    with pytest.raises(ConfigError):
        orc.tile_origins(100, 256, 26)


def test_partition_coverage(orc):  # test_parallel.cpp:151-168
    cfg = toy_cfg()
    t = orc.partition_tiles(170, 120, cfg, orc.led_sequence("spiral", cfg))
    assert len(t.xy) == 6
    cov = np.zeros((120, 170), int)
    for x0, y0 in t.xy:
        assert x0 + 64 <= 170 and y0 + 64 <= 120
        cov[y0:y0 + 64, x0:x0 + 64] += 1
    assert cov.min() >= 1
    assert t.kvecs[0, 0, 0] != t.kvecs[1, 0, 0]


def test_worker_invariance_and_extent(orc):  # test_parallel.cpp:170-200
    cfg = toy_cfg()
    up = cfg.upsample
    obj = orc.synth_object("composite", 120 * up, 31)[: 64 * up, : 120 * up]
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    assert (fs.width, fs.height) == (120, 64)
    a = orc.run_offline(fs, cfg, seq, 2, workers=1)
    b = orc.run_offline(fs, cfg, seq, 2, workers=4)
    assert a.tile_count == 2
    assert np.array_equal(a.tiles, b.tiles) and np.array_equal(a.stitched, b.stitched)
    full = orc.simulate_dataset(orc.synth_object("composite", 120 * up, 32), seq, cfg)
    r = orc.run_offline(full, cfg, seq, 1)
    assert r.stitched.shape == (120 * up, 120 * up)


# ---------------------------------------------------------------- test_stitch.cpp
def rand_stitch(rows, cols, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (rows, cols)) + 2.0 + 1j * rng.uniform(-1, 1, (rows, cols))


def test_mean_ratio_properties(orc):  # test_stitch.cpp:26-67
    f1, f2 = rand_stitch(16, 32, 7), rand_stitch(16, 32, 77)
    f2[:, :8] = f1[:, -8:]
    assert abs(orc.mean_ratio(f1, f2, 8) - 1) < 1e-14
    g = 0.5 * np.exp(1j * math.pi / 4)
    f2 = rand_stitch(16, 32, 9)
    f2[:, :8] = g * f1[:, -8:]
    r = orc.mean_ratio(f1, f2, 8)
    assert abs(r - 1 / g) < 1e-13 and abs(r) == pytest.approx(2.0)
    for seed in range(5):
        a, b = rand_stitch(20, 20, 100 + seed), rand_stitch(20, 20, 200 + seed)
        assert abs(orc.mean_ratio(a, b, 6) - a[:, -6:].mean() / b[:, :6].mean()) < 1e-13
        assert abs(orc.mean_ratio(a, b, 6, True) - a[-6:, :].mean() / b[:6, :].mean()) < 1e-13


def test_degenerate_overlap(orc):  # test_stitch.cpp:69-74
    with pytest.raises(DataError, match="degenerate overlap"):
        orc.mean_ratio(rand_stitch(8, 16, 3), np.zeros((8, 16), complex), 4)


def test_stitch_pair_486_and_reassembly(orc):  # test_stitch.cpp:76-98
    f1, f2 = rand_stitch(32, 256, 11), rand_stitch(32, 256, 12)
    f2[:, :26] = f1[:, -26:]
    assert orc.stitch_pair(f1, f2, 26).shape == (32, 486)
    whole = rand_stitch(24, 60, 13)
    out = orc.stitch_pair(whole[:, :34], whole[:, 26:], 8)
    assert np.abs(out - whole).max() < 1e-12
    g = 1.7 * np.exp(-0.9j)
    assert np.abs(orc.stitch_pair(whole[:, :34], g * whole[:, 26:], 8) - whole).max() < 1e-11


def test_stitch_transpose_and_zero_overlap(orc):  # test_stitch.cpp:100-117
    f1, f2 = rand_stitch(30, 14, 17), rand_stitch(30, 14, 18)
    v = orc.stitch_pair(f1, f2, 6, vertical=True)
    h = orc.stitch_pair(f1.T, f2.T, 6)
    assert v.shape == (54, 14) and np.array_equal(v, h.T)
    a, b = rand_stitch(10, 12, 19), rand_stitch(10, 8, 20)
    out = orc.stitch_pair(a, b, 0)
    assert np.array_equal(out[:, :12], a) and np.array_equal(out[:, 12:], b)


def test_mosaics(orc):  # test_stitch.cpp:128-178
    cfg = toy_cfg()
    up, fov = cfg.upsample, 120
    t = orc.partition_tiles(fov, fov, cfg, [cfg.center_led])
    whole = rand_stitch(fov * up, fov * up, 31)
    tiles = np.stack([whole[y * up:(y + 64) * up, x * up:(x + 64) * up] for x, y in t.xy])
    out = orc.stitch_mosaic(tiles, t.xy, cfg)
    assert out.shape == (fov * up, fov * up) and np.abs(out - whole).max() < 1e-11
    rng = np.random.default_rng(5)
    ph = np.exp(1j * rng.uniform(-math.pi, math.pi, len(t.xy)))
    out = orc.stitch_mosaic(tiles * ph[:, None, None], t.xy, cfg)
    g = tiles[0, 0, 0] * ph[0] / whole[0, 0]
    assert np.abs(out - g * whole).max() < 1e-10
    big = Optics(upsample=1)
    tb = orc.partition_tiles(946, 946, big, [big.center_led])
    assert len(tb.xy) == 16
    tiles = np.stack([rand_stitch(256, 256, int(x) * 977 + int(y)) for x, y in tb.xy])
    assert orc.stitch_mosaic(tiles, tb.xy, big).shape == (946, 946)


# ---------------------------------------------------------------- EPRY extension anchors
def test_epry_alpha1_beta0_equals_gs(orc):
    """EPRY with alpha=1, beta=0, |P|=1 on D reproduces update_step."""
    cfg = toy_cfg(led_scan_rows=5, led_scan_cols=5)
    obj = orc.synth_object("composite", cfg.hr_size, 41)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg, defocus_um=5.0)
    for defocus in (0.0, 5.0):
        a = orc.reconstruct_tile(fs, cfg, 2, seq, tile_defocus=defocus)
        b = orc.reconstruct_tile(fs, cfg, 2, seq, mode="epry", alpha=1.0, beta=0.0, tile_defocus=defocus)
        assert np.abs(a.hr - b.hr).max() / np.abs(a.hr).max() < 1e-12
        assert np.allclose(a.residuals, b.residuals, rtol=1e-12)


def test_epry_fixed_point(orc):
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 3)
    fs = orc.simulate_dataset(obj, [cfg.center_led], cfg)
    canvas = orc.init_canvas(fs, cfg)
    pupil, _ = orc.build_pupil(cfg, cfg.tile_size, 7.0)
    t = orc.partition_tiles(64, 64, cfg, [(32, 33)])
    kv = tuple(t.kvecs[0, 0])
    oy, ox = t.offsets[0, 0]
    n, N = cfg.tile_size, cfg.hr_size
    r0, c0 = N // 2 + oy - n // 2, N // 2 + ox - n // 2
    I = np.abs(orc.ifft2(canvas[r0:r0 + n, c0:c0 + n] * pupil)) ** 2
    before, pb = canvas.copy(), pupil.copy()
    res = orc.update_step_epry(canvas, I, kv, pupil, cfg)
    assert res <= 1e-12
    assert np.abs(before - canvas).max() / np.abs(before).max() <= 1e-10
    assert np.abs(pb - pupil).max() <= 1e-10


def test_epry_recovers_defocus(orc):
    """Data simulated with a 40 um defocus; EPRY started from the in-focus pupil
    must lower GS's final residual, reconstruct the band-limited truth with a
    clearly lower phase error, and move the pupil toward the true defocus pupil."""
    cfg = toy_cfg(led_scan_rows=7, led_scan_cols=7)
    obj = orc.synth_object("composite", cfg.hr_size, 12)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg, defocus_um=40.0)
    gs = orc.reconstruct_tile(fs, cfg, 8, seq)
    ep = orc.reconstruct_tile(fs, cfg, 8, seq, mode="epry")
    assert ep.residuals[-1] < 0.9 * gs.residuals[-1]
    truth = orc.band_limit(obj, orc.synthesized_na(cfg), cfg)
    q = lambda hr: orc.rmse(hr * orc.global_alignment(hr, truth), truth)
    assert q(ep.hr)[1] < 0.8 * q(gs.hr)[1]
    true_p, _ = orc.build_pupil(cfg, cfg.tile_size, 40.0)
    sup = np.abs(true_p) > 0
    corr = lambda p: abs(np.vdot(p[sup], true_p[sup])) / (np.linalg.norm(p[sup]) * np.linalg.norm(true_p[sup]))
    assert corr(ep.pupil) > corr(np.ones_like(true_p)) + 0.002


def test_epry_stable_on_wide_scans(orc):
    """Bright-field-only pupil steps keep EPRY as well-conditioned as GS on a
    15x15 scan of a 64 px tile (where dark-field pupil steps diverge)."""
    cfg = toy_cfg(led_scan_rows=15, led_scan_cols=15, tile_overlap=0)
    obj = orc.synth_object("composite", cfg.hr_size, 6)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg, defocus_um=20.0)
    a = orc.reconstruct_tile(fs, cfg, 10, seq, mode="epry")
    b = orc.reconstruct_tile(fs, cfg, 10, seq, mode="epry", tile_defocus=1e-5)
    assert np.all(a.residuals < 1.0)
    assert np.linalg.norm(a.hr - b.hr) / np.linalg.norm(a.hr) < 1e-6


def test_pipelined_refuses_epry(orc):
    cfg = toy_cfg()
    obj = orc.synth_object("composite", cfg.hr_size, 3)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    with pytest.raises(ConfigError, match="Gerchberg-Saxton"):
        orc.reconstruct_tile(fs, cfg, 1, seq, mode="epry", pipelined=True)
