"""GPU forward model (paper_2203_02507_b200.forward)
against the oracle's simulate_dataset (forward.cpp:172-282): same u16 frames.
The CPU cases run the same torch code on the host; the GPU cases add a
BASELINE-scale property check (simulate -> reconstruct -> compare)."""
import numpy as np
import pytest

import paper_2203_02507_b200 as fpm
from paper_2203_02507_b200.forward import simulate_dataset
from tests.helpers import amp_phase_rel, gpu_cfg, orc_cfg

CASES = [  # (tile, overlap, scan, fov, order, defocus)
    (64, 8, 3, 64, "spiral", 0.0),
    (64, 8, 5, 120, "spiral", 0.0),     # guard bands 0/32 -> 96-px crops, feathered overlap
    (64, 8, 5, 121, "raster", 12.0),    # clamped last tile, odd guard, defocus CTF
    (64, 0, 3, 128, "spiral", -5.0),
    (128, 26, 3, 230, "spiral", 0.0),
]


def _frames_match(got, ref):
    d = np.abs(got.astype(np.int64) - ref.astype(np.int64))
    return d.max() <= 1 and np.count_nonzero(d) <= max(1, d.size // 100000)


def _case(orc, tile, ov, scan, fov, order, dz, seed=3):
    cfg = gpu_cfg(tile_size=tile, tile_overlap=ov, led_scan_rows=scan, led_scan_cols=scan)
    oc = orc_cfg(cfg)
    size = max(fov * 4, 256)
    obj = orc.synth_object("composite", size, seed)[: fov * 4, : fov * 4]
    seq = orc.led_sequence(order, oc)
    return cfg, obj, seq, orc.simulate_dataset(obj, seq, oc, defocus_um=dz)


@pytest.mark.parametrize("case", CASES[:4])
def test_forward_model_matches_oracle_cpu(orc, case):
    cfg, obj, seq, ref = _case(orc, *case)
    got = simulate_dataset(obj, seq, cfg, defocus_um=case[5], device="cpu")
    assert got.images.shape == ref.images.shape
    assert _frames_match(got.images, ref.images)
    assert [tuple(x) for x in got.leds] == [tuple(x) for x in ref.leds]
    assert np.allclose(got.timestamps, ref.timestamps)


def test_forward_model_errors_cpu():
    cfg = gpu_cfg()
    with pytest.raises(fpm.DataError, match="multiple of upsample"):
        simulate_dataset(np.ones((258, 258), complex), [(32, 32)], cfg, device="cpu")
    with pytest.raises(fpm.DataError, match="identically zero"):
        simulate_dataset(np.zeros((256, 256), complex), [(32, 32)], cfg, device="cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_forward_model_matches_oracle_gpu(orc, case):
    cfg, obj, seq, ref = _case(orc, *case)
    got = simulate_dataset(obj, seq, cfg, defocus_um=case[5], device="cuda")
    assert _frames_match(got.images, ref.images)


@pytest.mark.gpu
def test_simulate_then_reconstruct_at_scale(orc):
    """A 512-px FOV (64 tiles, 15x15 LEDs, the config-3 tile geometry) simulated
    on the GPU, reconstructed on the GPU, against the oracle's reconstruction of
    the same frames (1e-3, the north star's full-count bound) and the truth."""
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=0, upsample=4, led_scan_rows=15, led_scan_cols=15)
    oc = orc_cfg(cfg)
    obj = orc.synth_object("composite", 2048, 11)
    seq = orc.led_sequence("spiral", oc)
    fs = simulate_dataset(obj, seq, cfg, device="cuda")
    assert fs.images.shape == (225, 512, 512)
    opt = fpm.RunOptions(iters=3)
    got = fpm.run_offline(fs, cfg, seq, opt, stitch=False)
    ofs = orc.FrameStack(fs.images, list(fs.leds))
    ref = orc.run_offline(ofs, oc, seq, 3, want_stitched=False, want_tiles=True)
    for t in (0, 27, 63):
        amp, ph = amp_phase_rel(got.tiles[t], ref.tiles[t])
        assert amp < 1e-3 and ph < 1e-3, (t, amp, ph)


@pytest.mark.gpu
def test_config3_full_fov_physical_parity(orc):
    """BASELINE config 3 at full size on physical data: a 2048x2048-sensor stack
    (1,024 tiles, 15x15 LEDs, per-tile defocus) simulated on the GPU,
    reconstructed with 10 EPRY iterations in one launch; a corner, an edge and an
    interior tile against the oracle's reconstruct_tile of the same frames
    (north-star check 3: <= 1e-3 after the full count)."""
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=0, upsample=4, led_scan_rows=15, led_scan_cols=15)
    oc = orc_cfg(cfg)
    obj = orc.synth_object("composite", 8192, 21)
    seq = orc.led_sequence("spiral", oc)
    fs = simulate_dataset(obj, seq, cfg, defocus_um=6.0, device="cuda")
    assert fs.images.shape == (225, 2048, 2048)
    T = 1024
    rng = np.random.default_rng(7)
    defocus = rng.uniform(-10, 10, T)
    opt = fpm.RunOptions(iters=10, mode="epry", tile_defocus_um=list(defocus))
    got = fpm.run_offline(fs, cfg, seq, opt, stitch=False)
    assert got.tiles.shape == (T, 256, 256)
    ofs = orc.FrameStack(fs.images, list(fs.leds))
    for t in (0, 31, 528):
        ref = orc.reconstruct_tile(ofs, oc, 10, seq, tile_index=t, mode="epry", tile_defocus=float(defocus[t]))
        amp, ph = amp_phase_rel(got.tiles[t], ref.hr)
        assert amp < 1e-3 and ph < 1e-3, (t, amp, ph)
        assert np.allclose(got.tile_metrics[t].pass_mean_residual, ref.residuals, rtol=1e-3)


@pytest.mark.gpu
def test_acceptance_round_trip_recovery_on_device(orc):
    """Acceptance criterion 1 (acceptance.cpp:99-121) on the device: stock
    geometry (256-px tile, upsample 4, 9x9 LEDs), composite object, 5 GS
    iterations; the globally aligned reconstruction against the band-limited
    truth must reach amplitude RMSE <= 0.03 and phase RMSE <= 0.1 rad."""
    cfg = fpm.OpticalConfig(led_scan_rows=9, led_scan_cols=9)
    oc = orc_cfg(cfg)
    obj = orc.synth_object("composite", 1024, 1)
    seq = orc.led_sequence("spiral", oc)
    fs = simulate_dataset(obj, seq, cfg, device="cuda")
    t = fpm.partition_tiles(fs.width(), fs.height(), cfg)[0]
    res = fpm.reconstruct_tile(fs, t, cfg, 5, seq)
    truth = orc.band_limit(obj, fpm.synthesized_na(cfg), oc)
    aligned = res.hr.astype(np.complex128) * orc.global_alignment(res.hr, truth)
    arms, prms = orc.rmse(aligned, truth)
    assert arms <= 0.03 and prms <= 0.1, (arms, prms)


def _bar_groups(size):
    """USAF-like bar groups of the Bars object (forward.cpp:22-40)."""
    out = []
    band = size // 5
    for g, p in enumerate((64, 32, 16, 8, 4)):
        start = size // 2 - (5 * p) // 4
        out.append(dict(period=p, row=(g * band + band // 4 + g * band + 3 * band // 4) // 2,
                        bars=[start + b * p + p // 4 for b in range(3)],
                        gaps=[start + b * p + (3 * p) // 4 for b in range(2)]))
    return out


def _min_resolved_period(amp, size, scale):
    """Smallest bar period with contrast >= 0.2 (acceptance.cpp:57-73)."""
    best = 1 << 20
    for g in _bar_groups(size):
        row = g["row"] // scale
        bar = np.mean([amp[row, x // scale] for x in g["bars"]])
        gap = np.mean([amp[row, x // scale] for x in g["gaps"]])
        if (gap - bar) / (gap + bar) >= 0.2:
            best = min(best, g["period"])
    return best


@pytest.mark.gpu
def test_acceptance_resolution_gain_on_device(orc):
    """Acceptance criterion 2 (acceptance.cpp:125-145) on the device: the Bars
    object under the stock 13x13 scan; the reconstruction (3 GS iterations)
    must resolve bars at most half the period the on-axis LR frame resolves."""
    cfg = fpm.OpticalConfig()
    oc = orc_cfg(cfg)
    obj = orc.synth_object("bars", 1024, 0)
    seq = orc.led_sequence("spiral", oc)
    fs = simulate_dataset(obj, seq, cfg, device="cuda")
    lr_amp = np.sqrt(fs.images[fs.find(cfg.center_led)].astype(np.float64))
    lr_min = _min_resolved_period(lr_amp, 1024, cfg.upsample)
    t = fpm.partition_tiles(fs.width(), fs.height(), cfg)[0]
    res = fpm.reconstruct_tile(fs, t, cfg, 3, seq)
    hr_min = _min_resolved_period(np.abs(res.hr), 1024, 1)
    assert lr_min < (1 << 20), "no bars resolved in the LR frame"
    assert 2 * hr_min <= lr_min, (lr_min, hr_min)


def _seam_phase_jump(f, seam, vertical):
    """Mean |wrapped phase step| across a seam (metrics.cpp:59-85)."""
    a = np.angle(f[:, seam]) - np.angle(f[:, seam - 1]) if vertical else \
        np.angle(f[seam, :]) - np.angle(f[seam - 1, :])
    return float(np.mean(np.abs((a + np.pi) % (2 * np.pi) - np.pi)))


@pytest.mark.gpu
def test_acceptance_stitch_continuity_on_device(orc):
    """Acceptance criterion 6 (acceptance.cpp:272-308) on the device: 2x2 tiles
    of 256 px, 5x5 LEDs, 3 iterations; the Eq. (1) mosaic with a 26-px overlap
    must cut the seam phase jump below 0.2x that of the overlap-free mosaic,
    and 256 + 256 - 26 = 486 must hold for the mosaic width."""
    def stitched_for(overlap, fov):
        cfg = fpm.OpticalConfig(led_scan_rows=5, led_scan_cols=5, tile_overlap=overlap)
        oc = orc_cfg(cfg)
        obj = orc.synth_object("composite", fov * cfg.upsample, 9)
        seq = orc.led_sequence("spiral", oc)
        fs = simulate_dataset(obj, seq, cfg, device="cuda")
        return fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=3)).stitched

    with_ov, no_ov = stitched_for(26, 486), stitched_for(0, 512)
    up = 4
    assert with_ov.shape == (486 * up, 486 * up)
    jump_ov = 0.5 * (_seam_phase_jump(with_ov, 243 * up, True) + _seam_phase_jump(with_ov, 243 * up, False))
    jump_no = 0.5 * (_seam_phase_jump(no_ov, 256 * up, True) + _seam_phase_jump(no_ov, 256 * up, False))
    assert jump_ov < 0.2 * jump_no, (jump_ov, jump_no)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(3, 96, 120), (2, 384, 480), (1, 512, 512), (5, 60, 75), (2, 1024, 2048)])
def test_fft2_c128_matches_numpy(shape):
    """The forward model's FP64 2-D FFT (fpmgpu_fft2_c128, radix 2/3/4/5) against
    numpy on the guard-banded tile sizes: forward and inverse to 1e-12 relative."""
    import torch
    from paper_2203_02507_b200.forward import fft2_c128
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    t = torch.from_numpy(x).cuda()
    for inverse, ref in ((False, np.fft.fft2(x)), (True, np.fft.ifft2(x))):
        got = fft2_c128(t, inverse).cpu().numpy()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12, (shape, inverse)


@pytest.mark.gpu
def test_fft2_c128_sizes_refused():
    """Sides with a prime factor above 5 have no kernel: UnsupportedError, not a fallback."""
    import torch
    from paper_2203_02507_b200.forward import fft2_c128
    with pytest.raises(fpm.UnsupportedError, match="factor into 2, 3 and 5"):
        fft2_c128(torch.zeros((2, 49, 64), dtype=torch.complex128, device="cuda"))
