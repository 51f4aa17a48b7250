"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Tolerances (north star, BASELINE.json): reconstructed amplitude and phase
within relative L2 1e-4 per iteration and 1e-3 after the full iteration
count. The kernel computes in FP32, the oracle in FP64.
"""
import numpy as np
import pytest

import paper_2203_02507_b200 as fpm
from tests.helpers import amp_phase_rel, dataset, gpu_cfg, orc_cfg, rel_l2

pytestmark = pytest.mark.gpu

PER_ITER_TOL = 1e-4
FINAL_TOL = 1e-3


def test_init_canvas_and_finalize(orc, eng):
    cfg = gpu_cfg()
    fs, ofs, seq, _ = dataset(cfg, seed=2)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    got = fpm.init_canvas(fs, t, cfg, engine=eng).spectrum
    ref = orc.init_canvas(ofs, orc_cfg(cfg))
    assert rel_l2(got, ref) < 1e-6
    back = fpm.canvas_to_field(fpm.SpectrumCanvas(got, cfg), engine=eng)
    ref_back = orc.canvas_to_field(ref, orc_cfg(cfg))
    assert rel_l2(back, ref_back) < 1e-6
    # zero iterations round trip (test_recon.cpp:77-86)
    expected = orc.upsample_bilinear(np.sqrt(fs.images[fs.find(cfg.center_led)].astype(float)), 4)
    assert np.abs(np.abs(back) - expected).max() / expected.max() < 1e-5


@pytest.mark.parametrize("defocus", [0.0, 9.0])
def test_update_step_matches_oracle(orc, eng, defocus):
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5)
    fs, ofs, seq, _ = dataset(cfg, seed=3)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    canvas = orc.init_canvas(ofs, orc_cfg(cfg))
    pupil = fpm.build_pupil(cfg, 64, defocus)
    for led in seq[:6]:
        I = fs.images[fs.find(led)][:64, :64].astype(np.float64)
        wv = t.wavevectors[led]
        gc = fpm.SpectrumCanvas(canvas.astype(np.complex64), cfg)
        r_gpu = fpm.update_step(gc, I, wv, pupil, engine=eng)
        r_ref = orc.update_step(canvas, I, wv, pupil.values, orc_cfg(cfg))
        assert r_gpu == pytest.approx(r_ref, rel=1e-4, abs=1e-9)
        assert rel_l2(gc.spectrum, canvas) < 1e-5


def test_update_step_fixed_point(orc, eng):
    """test_recon.cpp:96-116 on the device: self-consistent data is a fixed point."""
    cfg = gpu_cfg()
    fs, ofs, _, _ = dataset(cfg, seed=3)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    canvas = orc.init_canvas(ofs, orc_cfg(cfg))
    pupil = fpm.build_pupil(cfg, 64)
    wv = t.wavevectors[(32, 33)]
    oy, ox = fpm.spectrum_offset_px(wv, cfg)
    r0, c0 = 128 + oy - 32, 128 + ox - 32
    I = np.abs(orc.ifft2(canvas[r0:r0 + 64, c0:c0 + 64] * pupil.values)) ** 2
    gc = fpm.SpectrumCanvas(canvas.astype(np.complex64), cfg)
    res = fpm.update_step(gc, I, wv, pupil, engine=eng)
    assert res <= 1e-10
    assert np.abs(gc.spectrum - canvas).max() / np.abs(canvas).max() <= 1e-6


def test_support_confinement_bit_exact(orc, eng):
    """test_recon.cpp:118-145: pixels outside every updated disk are untouched."""
    cfg = gpu_cfg()
    fs, ofs, seq, _ = dataset(cfg, seed=4)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    init = fpm.init_canvas(fs, t, cfg, engine=eng)
    gc = fpm.SpectrumCanvas(init.spectrum.copy(), cfg)
    pupil = fpm.build_pupil(cfg, 64)
    for led in seq:
        fpm.update_step(gc, fs.images[fs.find(led)][:64, :64], t.wavevectors[led], pupil, engine=eng)
    N = 256
    i, j = np.mgrid[0:N, 0:N]
    inside = np.zeros((N, N), bool)
    for oy, ox in gc.updated_offsets:
        inside |= np.hypot(i - (N // 2 + oy), j - (N // 2 + ox)) <= pupil.radius_px
    assert np.array_equal(gc.spectrum[~inside], init.spectrum[~inside])


@pytest.mark.parametrize("iters", [1, 2, 5])
def test_gs_per_iteration(orc, eng, iters):
    """Config 1 geometry (64x64 LR, 15x15 LEDs, GS) per iteration count."""
    cfg = gpu_cfg(led_scan_rows=15, led_scan_cols=15, tile_overlap=0)
    fs, ofs, seq, _ = dataset(cfg, seed=1)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    got = fpm.reconstruct_tile(fs, t, cfg, iters, seq, engine=eng)
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), iters, seq)
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < PER_ITER_TOL and ph < PER_ITER_TOL, (amp, ph)
    assert np.allclose(got.metrics.pass_mean_residual, ref.residuals, rtol=1e-3)


def test_config1_full_gs(orc, eng):
    """BASELINE config 1: single 64x64 tile, 15x15 LEDs, 10 iterations GS."""
    cfg = gpu_cfg(led_scan_rows=15, led_scan_cols=15, tile_overlap=0)
    fs, ofs, seq, _ = dataset(cfg, seed=1)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    got = fpm.reconstruct_tile(fs, t, cfg, 10, seq, engine=eng)
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), 10, seq)
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < FINAL_TOL and ph < FINAL_TOL, (amp, ph)
    assert np.allclose(got.metrics.pass_mean_residual, ref.residuals, rtol=1e-3)


@pytest.mark.parametrize("iters", [1, 3])
def test_epry_per_iteration(orc, eng, iters):
    cfg = gpu_cfg(led_scan_rows=9, led_scan_cols=9, tile_overlap=0)
    fs, ofs, seq, _ = dataset(cfg, seed=5, defocus_um=25.0)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    got = fpm.reconstruct_tile(fs, t, cfg, iters, seq, mode="epry", engine=eng)
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), iters, seq, mode="epry")
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < PER_ITER_TOL and ph < PER_ITER_TOL, (amp, ph)
    assert rel_l2(got.pupil, ref.pupil) < PER_ITER_TOL


def test_epry_defocused_tile_final(orc, eng):
    cfg = gpu_cfg(led_scan_rows=15, led_scan_cols=15, tile_overlap=0)
    fs, ofs, seq, _ = dataset(cfg, seed=6, defocus_um=20.0)
    tiles = fpm.partition_tiles(64, 64, cfg)
    tiles[0].defocus_um = 5.0
    got = fpm.reconstruct_tile(fs, tiles[0], cfg, 10, seq, mode="epry", engine=eng)
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), 10, seq, mode="epry", tile_defocus=5.0)
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < FINAL_TOL and ph < FINAL_TOL, (amp, ph)


@pytest.mark.parametrize("n", [64, 128, 256])
def test_pipelined_bit_identical_to_sequential(eng, n):
    """Spectrum-domain level: pipelined == sequential bit for bit (test_parallel.cpp:79-122),
    on the lattice kernel (n = 64) and the general warp-FFT kernel (n = 128, 256)."""
    cfg = gpu_cfg(tile_size=n, led_scan_rows=7, led_scan_cols=7, tile_overlap=0)
    fs, _, _, _ = dataset(cfg, seed=23)
    seq = fpm.led_sequence("raster", cfg)
    t = fpm.partition_tiles(n, n, cfg)[0]
    lag = fpm.min_safe_lag_tile(seq, t, cfg)
    assert lag < len(seq)
    a = fpm.reconstruct_tile(fs, t, cfg, 3, seq, engine=eng)
    b = fpm.pipelined_reconstruct_tile(fs, t, cfg, 3, seq, lag=lag, engine=eng)
    assert b.lag == lag and not b.nondeterministic
    assert np.array_equal(a.hr, b.hr)
    c = fpm.pipelined_reconstruct_tile(fs, t, cfg, 3, seq, engine=eng)
    assert np.array_equal(a.hr, c.hr)


def test_unsafe_lag_refused(eng):
    cfg = gpu_cfg()
    fs, _, seq, _ = dataset(cfg, seed=24)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    with pytest.raises(fpm.UnsafeLagError) as ei:
        fpm.pipelined_reconstruct_tile(fs, t, cfg, 2, seq, lag=1, engine=eng)
    assert ei.value.minimum == 9
    f = fpm.pipelined_reconstruct_tile(fs, t, cfg, 2, seq, lag=1, force_unsafe=True, engine=eng)
    assert f.nondeterministic and np.all(np.isfinite(f.hr))


def test_multi_tile_batch_matches_oracle(orc, eng):
    """Spatial level: many tiles per launch, per-tile k-vectors and defocus pupils (config 3 shape, small FOV)."""
    cfg = gpu_cfg(led_scan_rows=7, led_scan_cols=7, tile_overlap=8)
    fs, ofs, seq, _ = dataset(cfg, fov=120, seed=31)
    rng = np.random.default_rng(7)
    defocus = rng.uniform(-10, 10, 4)
    opt = fpm.RunOptions(iters=3, mode="epry", tile_defocus_um=list(defocus))
    got = fpm.run_offline(fs, cfg, seq, opt, engine=eng, stitch=False)
    ref = orc.run_offline(ofs, orc_cfg(cfg), seq, 3, mode="epry", tile_defocus=defocus, want_stitched=False)
    assert got.tiles.shape == ref.tiles.shape == (4, 256, 256)
    for i in range(4):
        amp, ph = amp_phase_rel(got.tiles[i], ref.tiles[i])
        assert amp < FINAL_TOL and ph < FINAL_TOL, (i, amp, ph)


QUAD_DATA = {"gs": dict(rows=15, seed=1, defocus=0.0), "epry": dict(rows=9, seed=5, defocus=25.0)}


@pytest.mark.parametrize("mode,iters", [("gs", 1), ("gs", 2), ("gs", 10), ("epry", 1), ("epry", 3)])
@pytest.mark.parametrize("quad", ["0", "1"])
def test_n64_kernels_match_oracle(orc, eng, monkeypatch, mode, iters, quad):
    """n = 64 on the 128-thread pair lattice (kernels.cu) and on the 256-thread quad
    lattice (kernels_quad.cu), each forced, against the oracle: 1e-4 per iteration,
    1e-3 after the full count (config 1)."""
    monkeypatch.setenv("FPM_B200_QUAD", quad)
    d = QUAD_DATA[mode]
    cfg = gpu_cfg(led_scan_rows=d["rows"], led_scan_cols=d["rows"], tile_overlap=0)
    fs, ofs, seq, _ = dataset(cfg, seed=d["seed"], defocus_um=d["defocus"])
    t = fpm.partition_tiles(64, 64, cfg)[0]
    got = fpm.reconstruct_tile(fs, t, cfg, iters, seq, mode=mode, engine=fpm.Engine(0))
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), iters, seq, mode=mode)
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    tol = FINAL_TOL if iters == 10 else PER_ITER_TOL
    assert amp < tol and ph < tol, (amp, ph)
    assert np.allclose(got.metrics.pass_mean_residual, ref.residuals, rtol=1e-3)
    if mode == "epry":
        assert rel_l2(got.pupil, ref.pupil) < tol


@pytest.mark.parametrize("queue", ["0", "1"])
def test_quad_kernel_multi_tile_batch(orc, eng, monkeypatch, queue):
    """Per-tile k-vectors and defocus pupils on the quad-lattice kernel, one CTA
    per tile and as the work queue, against the oracle; the two schedules agree
    bit for bit."""
    monkeypatch.setenv("FPM_B200_QUAD", "1")
    monkeypatch.setenv("FPM_B200_BANDS", "1")
    cfg = gpu_cfg(led_scan_rows=7, led_scan_cols=7, tile_overlap=8)
    fs, ofs, seq, _ = dataset(cfg, fov=120, seed=31)
    rng = np.random.default_rng(7)
    defocus = rng.uniform(-10, 10, 4)
    opt = fpm.RunOptions(iters=3, mode="epry", tile_defocus_um=list(defocus))
    monkeypatch.setenv("FPM_B200_QUEUE", "0")
    a = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    monkeypatch.setenv("FPM_B200_QUEUE", queue)
    got = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    assert np.array_equal(a.tiles, got.tiles)
    assert np.array_equal(np.array([m.pass_mean_residual for m in a.tile_metrics]),
                          np.array([m.pass_mean_residual for m in got.tile_metrics]))
    ref = orc.run_offline(ofs, orc_cfg(cfg), seq, 3, mode="epry", tile_defocus=defocus, want_stitched=False)
    for i in range(4):
        amp, ph = amp_phase_rel(got.tiles[i], ref.tiles[i])
        assert amp < FINAL_TOL and ph < FINAL_TOL, (i, amp, ph)


def test_quad_kernel_agrees_with_pair_kernel(eng, monkeypatch):
    """The two n = 64 kernels compute the same reconstruction (different lane
    splits of the same factorisation: equal to FP32 rounding)."""
    cfg = gpu_cfg(led_scan_rows=9, led_scan_cols=9, tile_overlap=8)
    fs, _, seq, _ = dataset(cfg, fov=120, seed=33)
    opt = fpm.RunOptions(iters=2, mode="epry", tile_defocus_um=[3.0, -2.0, 0.0, 5.0])
    monkeypatch.setenv("FPM_B200_QUAD", "0")
    a = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    monkeypatch.setenv("FPM_B200_QUAD", "1")
    b = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    for i in range(4):
        assert rel_l2(b.tiles[i], a.tiles[i]) < 1e-5
        assert rel_l2(b.pupils[i], a.pupils[i]) < 1e-5


def test_offset_out_of_canvas_is_data_error(eng):
    cfg = gpu_cfg()
    fs, _, seq, _ = dataset(cfg, seed=2)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    canvas = fpm.init_canvas(fs, t, cfg, engine=eng)
    with pytest.raises(fpm.DataError, match="spectrum offset out of canvas bounds"):
        fpm.update_step(canvas, np.ones((64, 64)), (0.95 / cfg.wavelength, 0.0), fpm.build_pupil(cfg, 64),
                        engine=eng)


def _stitch_case(orc, cfg, fov, seed, phases=False):
    rng = np.random.default_rng(seed)
    up = cfg.upsample
    whole = (rng.uniform(-1, 1, (fov * up, fov * up)) + 2.0) + 1j * rng.uniform(-1, 1, (fov * up, fov * up))
    specs = fpm.partition_tiles(fov, fov, cfg)
    tiles = np.stack([whole[s.y0 * up:(s.y0 + cfg.tile_size) * up, s.x0 * up:(s.x0 + cfg.tile_size) * up]
                      for s in specs])
    if phases:
        tiles = tiles * np.exp(1j * rng.uniform(-np.pi, np.pi, len(specs)))[:, None, None]
    xy = np.array([[s.x0, s.y0] for s in specs], np.int32)
    return tiles, xy, specs


@pytest.mark.parametrize("fov,ov,phases", [(120, 8, False), (120, 8, True), (121, 8, True), (128, 0, False),
                                           (200, 24, True)])
def test_stitch_mosaic_matches_oracle(orc, eng, fov, ov, phases):
    """Eq. (1) mosaic on the device vs stitch_mosaic (stitch.cpp:48-86), incl. a clamped final tile."""
    cfg = gpu_cfg(tile_overlap=ov)
    tiles, xy, specs = _stitch_case(orc, cfg, fov, fov + ov, phases)
    got = fpm.stitch_mosaic(tiles.astype(np.complex64), specs, cfg, engine=eng)
    ref = orc.stitch_mosaic(tiles, xy, orc_cfg(cfg))
    assert got.shape == ref.shape == (fov * 4, fov * 4)
    assert rel_l2(got, ref) < 1e-5


def test_run_offline_stitched_matches_oracle(orc, eng):
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=8)
    fs, ofs, seq, _ = dataset(cfg, fov=120, seed=32)
    got = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=2), engine=eng)
    ref = orc.run_offline(ofs, orc_cfg(cfg), seq, 2)
    assert got.stitched.shape == ref.stitched.shape == (480, 480)
    amp, ph = amp_phase_rel(got.stitched, ref.stitched)
    assert amp < 1e-4 and ph < 1e-4, (amp, ph)


# ---------------------------------------------------------------- n = 128 / 256 (box kernel)
def _single_tile(n, scan, seed, defocus=0.0):
    cfg = fpm.OpticalConfig(tile_size=n, tile_overlap=0, upsample=4, led_scan_rows=scan, led_scan_cols=scan)
    fs, ofs, seq, _ = dataset(cfg, seed=seed, defocus_um=defocus)
    return cfg, fs, ofs, seq, fpm.partition_tiles(n, n, cfg)[0]


@pytest.mark.parametrize("mode,iters", [("gs", 1), ("epry", 1), ("epry", 2)])
def test_n128_per_iteration(orc, eng, mode, iters):
    """Config 2 geometry (128x128 LR, 15x15 LEDs) per iteration, GS and EPRY."""
    cfg, fs, ofs, seq, t = _single_tile(128, 15, seed=2, defocus=15.0)
    got = fpm.reconstruct_tile(fs, t, cfg, iters, seq, mode=mode, engine=eng)
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), iters, seq, mode=mode)
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < PER_ITER_TOL and ph < PER_ITER_TOL, (amp, ph)
    assert np.allclose(got.metrics.pass_mean_residual, ref.residuals, rtol=1e-3)


def test_config2_full_epry(orc, eng):
    """BASELINE config 2: single 128x128 tile, 15x15 LEDs, EPRY, 20 iterations."""
    cfg, fs, ofs, seq, t = _single_tile(128, 15, seed=1, defocus=15.0)
    got = fpm.reconstruct_tile(fs, t, cfg, 20, seq, mode="epry", engine=eng)
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), 20, seq, mode="epry")
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < FINAL_TOL and ph < FINAL_TOL, (amp, ph)
    assert rel_l2(got.pupil, ref.pupil) < FINAL_TOL


@pytest.mark.parametrize("mode", ["gs", "epry"])
def test_n256_config5_geometry(orc, eng, mode):
    """Config 5 tile geometry: 256x256 LR (N = 1024), 21x21 LEDs."""
    cfg, fs, ofs, seq, t = _single_tile(256, 21, seed=5, defocus=10.0)
    got = fpm.reconstruct_tile(fs, t, cfg, 2, seq, mode=mode, engine=eng)
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), 2, seq, mode=mode)
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < PER_ITER_TOL and ph < PER_ITER_TOL, (amp, ph)
    assert np.allclose(got.metrics.pass_mean_residual, ref.residuals, rtol=1e-3)


@pytest.mark.parametrize("n", [128, 256])
def test_update_step_box_matches_oracle(orc, eng, n):
    cfg, fs, ofs, seq, t = _single_tile(n, 5, seed=7)
    canvas = orc.init_canvas(ofs, orc_cfg(cfg))
    pupil = fpm.build_pupil(cfg, n, 6.0)
    for led in seq[:4]:
        I = fs.images[fs.find(led)].astype(np.float64)
        gc = fpm.SpectrumCanvas(canvas.astype(np.complex64), cfg)
        r_gpu = fpm.update_step(gc, I, t.wavevectors[led], pupil, engine=eng)
        r_ref = orc.update_step(canvas, I, t.wavevectors[led], pupil.values, orc_cfg(cfg))
        assert r_gpu == pytest.approx(r_ref, rel=1e-4, abs=1e-9)
        assert rel_l2(gc.spectrum, canvas) < 1e-5


def test_box_kernel_agrees_with_lattice_kernel_n64(eng, monkeypatch):
    """The general warp-FFT kernel and the n = 64 lattice kernel compute the same update."""
    cfg = gpu_cfg(led_scan_rows=9, led_scan_cols=9, tile_overlap=8)
    fs, _, seq, _ = dataset(cfg, fov=120, seed=33)
    opt = fpm.RunOptions(iters=2, mode="epry", tile_defocus_um=[3.0, -2.0, 0.0, 5.0])
    a = fpm.run_offline(fs, cfg, seq, opt, engine=eng, stitch=False)
    monkeypatch.setenv("FPM_B200_FORCE_BOX", "1")
    b = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    for i in range(4):
        assert rel_l2(b.tiles[i], a.tiles[i]) < 1e-5


@pytest.mark.parametrize("bands", ["3", "16"])
def test_banded_host_path_bit_identical(eng, monkeypatch, bands):
    """The host path's row-band pipeline (H2D of band b+1 under the compute of
    band b) changes only the schedule: tiles, residuals and pupils are
    bit-identical to one unbanded launch."""
    cfg = gpu_cfg(led_scan_rows=7, led_scan_cols=7, tile_overlap=8)
    fs, _, seq, _ = dataset(cfg, fov=232, seed=34)
    specs = fpm.partition_tiles(fs.width(), fs.height(), cfg)
    rng = np.random.default_rng(3)
    opt = fpm.RunOptions(iters=2, mode="epry", tile_defocus_um=list(rng.uniform(-8, 8, len(specs))))
    monkeypatch.setenv("FPM_B200_BANDS", "1")
    a = fpm.run_offline(fs, cfg, seq, opt, engine=eng, stitch=False)
    monkeypatch.setenv("FPM_B200_BANDS", bands)
    b = fpm.run_offline(fs, cfg, seq, opt, engine=eng, stitch=False)
    assert len(specs) == 16
    assert np.array_equal(a.tiles, b.tiles)
    assert np.array_equal(np.array([m.pass_mean_residual for m in a.tile_metrics]),
                          np.array([m.pass_mean_residual for m in b.tile_metrics]))
    assert a.pupils is not None
    for pa, pb in zip(a.pupils, b.pupils):
        assert np.array_equal(pa, pb)


@pytest.mark.parametrize("mode,parts", [("gs", "1"), ("epry", "3"), ("epry", "")])
def test_work_queue_bit_identical(eng, monkeypatch, mode, parts):
    """The n = 64 LED loop as a persistent work queue over (pass, part, tile)
    items (FPM_B200_QUEUE=1 forces it, with a grid wider than the tile count, so
    most items wait on their tile's previous part held by another CTA) gives the
    one-CTA-per-tile launch's tiles, residuals and pupils bit for bit."""
    monkeypatch.setenv("FPM_B200_PARTS", parts)
    cfg = gpu_cfg(led_scan_rows=7, led_scan_cols=7, tile_overlap=8)
    fs, _, seq, _ = dataset(cfg, fov=232, seed=35)
    specs = fpm.partition_tiles(fs.width(), fs.height(), cfg)
    rng = np.random.default_rng(5)
    opt = fpm.RunOptions(iters=3, mode=mode, tile_defocus_um=list(rng.uniform(-8, 8, len(specs))))
    monkeypatch.setenv("FPM_B200_BANDS", "1")
    monkeypatch.setenv("FPM_B200_QUEUE", "0")
    a = fpm.run_offline(fs, cfg, seq, opt, engine=eng, stitch=False)
    monkeypatch.setenv("FPM_B200_QUEUE", "1")
    b = fpm.run_offline(fs, cfg, seq, opt, engine=eng, stitch=False)
    assert len(specs) == 16
    assert np.array_equal(a.tiles, b.tiles)
    assert np.array_equal(np.array([m.pass_mean_residual for m in a.tile_metrics]),
                          np.array([m.pass_mean_residual for m in b.tile_metrics]))
    if mode == "epry":
        for pa, pb in zip(a.pupils, b.pupils):
            assert np.array_equal(pa, pb)


@pytest.mark.parametrize("n,mode", [(256, "epry"), (128, "gs")])
def test_cluster_work_queue_bit_identical(eng, monkeypatch, n, mode):
    """The cluster kernel as a persistent work queue over (pass, tile) items
    (FPM_B200_QUEUE=1: a grid of clusters wider than the tile count, most items
    waiting on their tile's previous pass) gives one cluster per tile's bits."""
    cfg = fpm.OpticalConfig(tile_size=n, tile_overlap=0, upsample=4, led_scan_rows=5, led_scan_cols=5)
    fs, _, seq, _ = dataset(cfg, fov=2 * n, seed=42, defocus_um=4.0)
    specs = fpm.partition_tiles(fs.width(), fs.height(), cfg)
    opt = fpm.RunOptions(iters=3, mode=mode, tile_defocus_um=[2.0, -3.0, 0.0, 4.0][: len(specs)])
    monkeypatch.setenv("FPM_B200_BANDS", "1")
    monkeypatch.setenv("FPM_B200_CLUSTER", "4")
    monkeypatch.setenv("FPM_B200_QUEUE", "0")
    a = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    monkeypatch.setenv("FPM_B200_QUEUE", "1")
    b = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    assert len(specs) == 4
    assert np.array_equal(a.tiles, b.tiles)
    assert np.array_equal(np.array([m.pass_mean_residual for m in a.tile_metrics]),
                          np.array([m.pass_mean_residual for m in b.tile_metrics]))
    if mode == "epry":
        for pa, pb in zip(a.pupils, b.pupils):
            assert np.array_equal(pa, pb)


@pytest.mark.parametrize("n,cl,mode", [(128, 2, "epry"), (128, 4, "gs"), (128, 8, "epry"), (128, 16, "gs"), (256, 2, "gs"),
                                       (256, 4, "epry"), (256, 8, "gs")])
def test_cluster_kernel_matches_box_kernel(eng, monkeypatch, n, cl, mode):
    """A tile split over a CTA cluster (DSMEM column slabs) runs the box kernel's
    arithmetic element for element: same canvas bits, same pupil bits."""
    cfg = fpm.OpticalConfig(tile_size=n, tile_overlap=0, upsample=4, led_scan_rows=5, led_scan_cols=5)
    fs, _, seq, _ = dataset(cfg, seed=40, defocus_um=6.0)
    t = fpm.partition_tiles(n, n, cfg)[0]
    t.defocus_um = 4.0
    monkeypatch.setenv("FPM_B200_CLUSTER", "1")
    a = fpm.reconstruct_tile(fs, t, cfg, 2, seq, mode=mode, engine=fpm.Engine(0))
    monkeypatch.setenv("FPM_B200_CLUSTER", str(cl))
    b = fpm.reconstruct_tile(fs, t, cfg, 2, seq, mode=mode, engine=fpm.Engine(0))
    assert np.array_equal(a.hr, b.hr)
    if mode == "epry":
        assert np.array_equal(a.pupil, b.pupil)
    assert np.allclose(a.metrics.pass_mean_residual, b.metrics.pass_mean_residual, rtol=1e-5)


@pytest.mark.parametrize("cl,mode", [("1", "epry"), ("4", "epry"), ("4", "gs")])
def test_n256_box_pruning_matches_full_transforms(eng, monkeypatch, cl, mode):
    """WarpFFT256 with the support box inside [64, 192) skips the natural-layout
    registers 0, 1, 6, 7 (pruned first / last DFT8, no loads or stores for them);
    FPM_B200_MID=0 runs the full transforms. The two agree to FP32 rounding of
    signed zeros (bit for bit in practice)."""
    cfg = fpm.OpticalConfig(tile_size=256, tile_overlap=0, upsample=4, led_scan_rows=5, led_scan_cols=5)
    fs, _, seq, _ = dataset(cfg, seed=43, defocus_um=6.0)
    t = fpm.partition_tiles(256, 256, cfg)[0]
    t.defocus_um = 3.0
    monkeypatch.setenv("FPM_B200_CLUSTER", cl)
    monkeypatch.setenv("FPM_B200_MID", "0")
    a = fpm.reconstruct_tile(fs, t, cfg, 2, seq, mode=mode, engine=fpm.Engine(0))
    monkeypatch.delenv("FPM_B200_MID")
    b = fpm.reconstruct_tile(fs, t, cfg, 2, seq, mode=mode, engine=fpm.Engine(0))
    scale = np.abs(a.hr).max()
    assert np.abs(a.hr - b.hr).max() <= 1e-6 * scale
    assert np.allclose(a.metrics.pass_mean_residual, b.metrics.pass_mean_residual, rtol=1e-6)


@pytest.mark.parametrize("cl", [4, 8])
def test_cluster_kernel_n64_matches_oracle(orc, eng, monkeypatch, cl):
    """n = 64 on the cluster kernel (single-tile latency path) against the oracle."""
    cfg = gpu_cfg(led_scan_rows=7, led_scan_cols=7)
    fs, ofs, seq, _ = dataset(cfg, seed=41)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    monkeypatch.setenv("FPM_B200_CLUSTER", str(cl))
    got = fpm.reconstruct_tile(fs, t, cfg, 2, seq, mode="epry", engine=fpm.Engine(0))
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), 2, seq, mode="epry")
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < PER_ITER_TOL and ph < PER_ITER_TOL, (amp, ph)
    assert np.allclose(got.metrics.pass_mean_residual, ref.residuals, rtol=1e-3)


def test_async_requests_equal_sync(eng):
    """fpmgpu_reconstruct_tiles_async: three requests in flight back to back (the
    third waits for the first slot) give the synchronous call's bits."""
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=8)
    sets = [dataset(cfg, fov=120, seed=50 + k)[0] for k in range(3)]
    specs = fpm.partition_tiles(120, 120, cfg)
    seq = fpm.led_sequence("spiral", cfg)
    reqs = [fpm.make_request(fs, cfg, seq, specs, 2, mode="epry") for fs in sets]
    sync = [fpm.reconstruct_request(r, fs, eng) for r, fs in zip(reqs, sets)]
    pend = [fpm.reconstruct_request_async(r, fs, eng) for r, fs in zip(reqs, sets)]
    for p, ref in zip(pend, sync):
        hr, res, pup, _ = p.wait()
        assert np.array_equal(hr, ref[0]) and np.array_equal(res, ref[1]) and np.array_equal(pup, ref[2])


def _rect_dataset(cfg, h, w, seed, order="spiral", defocus=0.0, noise=None):
    from tests.helpers import orc
    oc = orc_cfg(cfg)
    size = max(h, w) * cfg.upsample
    obj = orc.synth_object("composite", max(size, 256), seed)[: h * cfg.upsample, : w * cfg.upsample]
    seq = orc.led_sequence(order, oc)
    fs = orc.simulate_dataset(obj, seq, oc, noise=noise, defocus_um=defocus)
    return fpm.FrameSet(fs.images, list(fs.leds), fs.timestamps), fs, seq


def test_rectangular_fov_with_clamped_tiles(orc):
    """Non-square FOV (120 x 184 LR px, overlap 8): clamped last tiles on both
    axes, raster order, EPRY with per-tile defocus; tiles and Eq. (1) mosaic
    against the oracle."""
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=8)
    fs, ofs, seq = _rect_dataset(cfg, 120, 184, seed=60, order="raster", defocus=4.0)
    specs = fpm.partition_tiles(184, 120, cfg)
    assert len(specs) == 2 * 4  # x: 0, 56, 112, 120 (clamped); y: 0, 56
    dz = np.linspace(-6, 6, len(specs))
    opt = fpm.RunOptions(iters=3, mode="epry", tile_defocus_um=list(dz))
    got = fpm.run_offline(fs, cfg, seq, opt)
    ref = orc.run_offline(ofs, orc_cfg(cfg), seq, 3, mode="epry", tile_defocus=dz)
    assert got.stitched.shape == ref.stitched.shape == (480, 736)
    for i in range(len(specs)):
        amp, ph = amp_phase_rel(got.tiles[i], ref.tiles[i])
        assert amp < FINAL_TOL and ph < FINAL_TOL, (i, amp, ph)
    amp, ph = amp_phase_rel(got.stitched, ref.stitched)
    assert amp < FINAL_TOL and ph < FINAL_TOL, (amp, ph)


def test_noisy_stack_and_upsample_8(orc):
    """Photon-noise frames (the reference's Poisson model) and a finer HR grid
    (upsample 8: N = 512 canvases for 64-px tiles) through the lattice kernel."""
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=0, upsample=8)
    fs, ofs, seq = _rect_dataset(cfg, 64, 64, seed=61, noise=(2000.0, 7))
    t = fpm.partition_tiles(64, 64, cfg)[0]
    got = fpm.reconstruct_tile(fs, t, cfg, 2, seq, mode="gs")
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), 2, seq, mode="gs")
    assert got.hr.shape == (512, 512)
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < PER_ITER_TOL and ph < PER_ITER_TOL, (amp, ph)
    assert np.allclose(got.metrics.pass_mean_residual, ref.residuals, rtol=1e-3)


def test_seed_frame_missing_uses_brightest(orc, capsys):
    """No on-axis frame: init_canvas seeds from the brightest frame with the
    reference's warning (recon.cpp:64-75); results still match the oracle."""
    cfg = gpu_cfg(led_scan_rows=3, led_scan_cols=3)
    fs, ofs, seq, _ = dataset(cfg, seed=62)
    keep = [k for k, led in enumerate(fs.leds) if tuple(led) != cfg.center_led]
    fs2 = fpm.FrameSet(fs.images[keep], [fs.leds[k] for k in keep])
    ofs2 = orc.FrameStack(fs.images[keep], [fs.leds[k] for k in keep])
    seq2 = [s for s in seq if tuple(s) != cfg.center_led]
    t = fpm.partition_tiles(64, 64, cfg)[0]
    got = fpm.reconstruct_tile(fs2, t, cfg, 2, seq2)
    assert "brightest frame" in capsys.readouterr().err
    ref = orc.reconstruct_tile(ofs2, orc_cfg(cfg), 2, seq2)
    amp, ph = amp_phase_rel(got.hr, ref.hr)
    assert amp < PER_ITER_TOL and ph < PER_ITER_TOL, (amp, ph)


def test_acceptance_criterion_7_format_hermeticity(tmp_path, eng):
    """acceptance.cpp:311-359 through the formats module: a dataset directory
    (frames/led_RR_CC.pgm + manifest.json) is read back and reconstructed twice;
    the CFI outputs (4 tiles + the stitched mosaic) are bit-identical across the
    runs, and CFI / PGM round trips are bit-exact."""
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=8, upsample=4, led_scan_rows=3, led_scan_cols=3)
    fs, _, seq, obj = dataset(cfg, fov=120, seed=7)
    fpm.write_dataset(tmp_path / "data", fs, cfg, object_truth=obj)
    outs = {}
    for run in ("run1", "run2"):
        ds = fpm.read_dataset(tmp_path / "data")
        res = fpm.run_offline(ds.frames, ds.cfg, fpm.led_sequence("spiral", ds.cfg), fpm.RunOptions(iters=2),
                              engine=eng)
        d = tmp_path / run
        d.mkdir()
        for i, t in enumerate(res.tiles):
            fpm.write_cfi(d / f"tile_{i:03d}.cfi", t)
        fpm.write_cfi(d / "stitched.cfi", res.stitched)
        outs[run] = sorted(p.name for p in d.iterdir() if p.suffix == ".cfi")
    assert outs["run1"] == outs["run2"] and len(outs["run1"]) >= 5
    for name in outs["run1"]:
        assert (tmp_path / "run1" / name).read_bytes() == (tmp_path / "run2" / name).read_bytes()
    fpm.write_cfi(tmp_path / "rt.cfi", fpm.read_cfi(tmp_path / "run1" / "stitched.cfi"))
    assert (tmp_path / "rt.cfi").read_bytes() == (tmp_path / "run1" / "stitched.cfi").read_bytes()
    pgm = tmp_path / "data" / "frames" / "led_32_32.pgm"
    fpm.write_pgm16(tmp_path / "rt.pgm", fpm.read_pgm16(pgm))
    assert (tmp_path / "rt.pgm").read_bytes() == pgm.read_bytes()


def test_acceptance_criterion_4_worker_and_batch_invariance(eng):
    """acceptance.cpp:176-246 (a) on the device: the 16 tiles of a 232-px FOV are
    identical for every worker count and for every batch size (max_tiles 4, 8,
    12, 16 reconstruct the leading tiles of the same partition) — tiles share
    nothing, and batch size only changes the kernel's schedule / build."""
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=8)
    fs, _, seq, _ = dataset(cfg, fov=232, seed=3)
    ref = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=1, workers=1, max_tiles=16), engine=eng, stitch=False)
    assert len(ref.tiles) == 16
    for w in (2, 4, 8):
        r = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=1, workers=w, max_tiles=16), engine=eng, stitch=False)
        assert np.array_equal(r.tiles, ref.tiles)
    for m in (4, 8, 12):
        r = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=1, max_tiles=m), engine=eng, stitch=False)
        assert np.array_equal(r.tiles, ref.tiles[:m])


@pytest.mark.parametrize("world", [2, 3])
def test_strong_scaling_bands_bit_identical(eng, world):
    """The strong-scaled data path (config 4/5) on one device: each rank's
    tile-row band (distributed.shard_request: its tiles, y-shifted, over its
    crop of the LR rows) reconstructs to the full FOV's tiles bit for bit."""
    from paper_2203_02507_b200.distributed import shard_request
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=8)
    fs, _, seq, _ = dataset(cfg, fov=176, seed=39)
    tiles = fpm.partition_tiles(fs.width(), fs.height(), cfg)
    for t, d in zip(tiles, np.random.default_rng(9).uniform(-8, 8, len(tiles))):
        t.defocus_um = float(d)
    full = fpm.make_request(fs, cfg, seq, tiles, 2, mode="epry")
    assert len(tiles) >= 3 * world
    hr_full, res_full, _, _ = fpm.reconstruct_request(full, fs, engine=eng)
    for r in range(world):
        me = shard_request(full, r, world)
        band = fpm.FrameSet(np.ascontiguousarray(fs.images[:, me.y_lo:me.y_hi, :]), fs.leds, fs.timestamps)
        hr, res, _, _ = fpm.reconstruct_request(me.request, band, engine=eng)
        assert np.array_equal(hr, hr_full[me.tiles])
        assert np.array_equal(res, res_full[me.tiles])
