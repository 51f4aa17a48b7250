"""Data formats: the reference's PGM16 / CFI / view /
config-JSON / dataset-directory readers and writers, re-expressed from its
`tests/test_io.cpp` (each case cites its line) plus a dataset round trip.
CPU only (the GPU acceptance criterion 7 is in test_gpu_parity.py)."""
import json
import math
import os

import numpy as np
import pytest

import paper_2203_02507_b200 as fpm
from paper_2203_02507_b200 import formats


def slurp(p):
    with open(p, "rb") as f:
        return f.read()


def test_pgm_bytes(tmp_path):  # test_io.cpp:36-48
    img = np.array([[0, 1], [65535, 256]], np.uint16)
    p = tmp_path / "t.pgm"
    fpm.write_pgm16(p, img)
    b = slurp(p)
    header = b"P5\n2 2\n65535\n"
    assert len(b) == len(header) + 8 and b.startswith(header)
    assert b[len(header):] == bytes([0x00, 0x00, 0x00, 0x01, 0xFF, 0xFF, 0x01, 0x00])


def test_pgm_round_trip_bit_exact(tmp_path):  # test_io.cpp:50-59
    img = np.random.default_rng(4).integers(0, 65536, (13, 7), dtype=np.uint16)
    p = tmp_path / "r.pgm"
    fpm.write_pgm16(p, img)
    back = fpm.read_pgm16(p)
    assert back.dtype == np.uint16 and np.array_equal(back, img)
    fpm.write_pgm16(tmp_path / "r2.pgm", back)
    assert slurp(p) == slurp(tmp_path / "r2.pgm")


def test_pgm_reader_rejects(tmp_path):  # test_io.cpp:61-77
    p = tmp_path / "bad.pgm"
    fpm.write_pgm16(p, np.full((4, 4), 9, np.uint16))
    os.truncate(p, os.path.getsize(p) - 1)
    with pytest.raises(fpm.IoError, match="expected 32 bytes, got 31"):
        fpm.read_pgm16(p)
    (tmp_path / "magic.pgm").write_text("P2\n2 2\n65535\n0 0 0 0\n")
    with pytest.raises(fpm.IoError, match="not a binary PGM"):
        fpm.read_pgm16(tmp_path / "magic.pgm")
    (tmp_path / "maxval.pgm").write_bytes(b"P5\n1 1\n255\n\0\0")
    with pytest.raises(fpm.IoError, match="maxval must be 65535"):
        fpm.read_pgm16(tmp_path / "maxval.pgm")
    with pytest.raises(fpm.IoError):
        fpm.read_pgm16(tmp_path / "absent.pgm")


def test_cfi_layout(tmp_path):  # test_io.cpp:79-97
    p = tmp_path / "one.cfi"
    fpm.write_cfi(p, np.array([[1.0 - 2.0j]]))
    b = slurp(p)
    assert len(b) == 28 and b[:4] == b"CFI1"
    assert b[4] == 1 and b[5] == 0 and b[8] == 1
    assert b[18] == 0xF0 and b[19] == 0x3F and b[27] == 0xC0


def test_cfi_round_trip_bit_exact(tmp_path):  # test_io.cpp:99-112
    rng = np.random.default_rng(5)
    f = rng.normal(size=(9, 17)) + 1j * rng.normal(size=(9, 17))
    f[0, 0] = complex(-0.0, 5e-324)  # signed zero and a subnormal keep their bits
    p = tmp_path / "rt.cfi"
    fpm.write_cfi(p, f)
    back = fpm.read_cfi(p)
    assert back.shape == (9, 17)
    assert back.view(np.uint64).tobytes() == f.view(np.uint64).tobytes()
    fpm.write_cfi(tmp_path / "rt2.cfi", back)
    assert slurp(p) == slurp(tmp_path / "rt2.cfi")


def test_cfi_refuses_non_finite_and_bad_magic(tmp_path):  # test_io.cpp:114-123
    f = np.zeros((3, 3), complex)
    f[2, 1] = complex(0.0, float("nan"))
    with pytest.raises(fpm.IoError, match=r"non-finite value at pixel \(2,1\)"):
        fpm.write_cfi(tmp_path / "nan.cfi", f)
    (tmp_path / "junk.cfi").write_bytes(b"NOPE")
    with pytest.raises(fpm.IoError, match="bad CFI magic"):
        fpm.read_cfi(tmp_path / "junk.cfi")
    fpm.write_cfi(tmp_path / "short.cfi", np.ones((2, 2)))
    os.truncate(tmp_path / "short.cfi", 20)
    with pytest.raises(fpm.IoError, match="unexpected end of file"):
        fpm.read_cfi(tmp_path / "short.cfi")


def test_amplitude_view_round_trip(tmp_path):  # test_io.cpp:125-137
    rng = np.random.default_rng(6)
    f = rng.uniform(0, 3, (12, 12)) * np.exp(1j * (rng.uniform(0, 3, (12, 12)) - 1.5))
    p = tmp_path / "amp.pgm"
    fpm.export_view(f, "amplitude", p)
    amp = fpm.import_view(p)
    step = np.abs(f).max() / 65535.0
    assert np.abs(amp - np.abs(f)).max() <= 0.5 * step * 1.0001


def test_phase_view_round_trip(tmp_path):  # test_io.cpp:139-152
    k = np.arange(64).reshape(8, 8)
    f = np.exp(1j * (-math.pi + 2 * math.pi * k / 64.0))
    p = tmp_path / "ph.pgm"
    fpm.export_view(f, "phase", p)
    ph = fpm.import_view(p)
    assert np.abs(ph - np.angle(f)).max() <= 0.5 * (2 * math.pi / 65535.0) * 1.0001


def test_zero_field_view(tmp_path):  # test_io.cpp:154-160
    p = tmp_path / "zero.pgm"
    fpm.export_view(np.zeros((4, 4), complex), "amplitude", p)
    assert np.all(fpm.read_pgm16(p) == 0)


def test_config_round_trip():  # test_io.cpp:162-182
    cfg = fpm.AppConfig()
    cfg.optics.tile_size, cfg.optics.tile_overlap = 128, 16
    cfg.run.iters, cfg.run.lag = 7, 3
    cfg.run.noise.enabled, cfg.run.noise.seed = True, 99
    back = fpm.config_from_json(fpm.config_to_json(cfg))
    assert back.optics.tile_size == 128 and back.optics.tile_overlap == 16
    assert back.optics.wavelength == cfg.optics.wavelength
    assert back.run.iters == 7 and back.run.lag == 3
    assert back.run.noise.enabled and back.run.noise.seed == 99
    assert fpm.config_from_json(fpm.config_to_json(fpm.AppConfig())).run.lag is None
    # defaults are materialised on write: every key present
    j = json.loads(fpm.config_to_json(fpm.AppConfig()))
    assert set(j["optics"]) == set(formats._OPTICS_KEYS) and set(j["run"]) == set(formats._RUN_KEYS)
    assert j["run"]["lag"] == "auto"


def test_config_rejects_unknown_keys():  # test_io.cpp:184-194
    for text, key in [('{"optics": {}, "runs": {}}', "runs"), ('{"optics": {"wavelength_nm": 525}}', "wavelength_nm"),
                      ('{"run": {"iterations": 5}}', "iterations"), ('{"run": {"noise": {"sigma": 1}}}', "sigma")]:
        with pytest.raises(fpm.ConfigError, match=f'unknown key "{key}"'):
            fpm.config_from_json(text)
    with pytest.raises(fpm.ConfigError):
        fpm.config_from_json("not json")


def test_config_rejects_invalid_values():  # test_io.cpp:196-202
    for text in ['{"optics": {"tile_overlap_px": 300}}', '{"optics": {"objective_na": -0.1}}', '{"run": {"iters": 0}}',
                 '{"run": {"order": "zigzag"}}', '{"run": {"mode": "batch"}}']:
        with pytest.raises(fpm.ConfigError):
            fpm.config_from_json(text)


def test_empty_config_is_stock():  # test_io.cpp:204-214
    cfg = fpm.config_from_json("{}")
    assert cfg.optics.wavelength == pytest.approx(0.525) and cfg.optics.objective_na == pytest.approx(0.1)
    assert cfg.optics.tile_size == 256 and cfg.optics.tile_overlap == 26 and cfg.optics.led_grid_rows == 64
    assert cfg.run.iters == 5 and cfg.run.order == "spiral" and cfg.run.mode == "offline"


def test_config_file_round_trip(tmp_path):
    cfg = fpm.AppConfig()
    cfg.optics.led_scan_rows = cfg.optics.led_scan_cols = 5
    fpm.write_config(tmp_path / "c.json", cfg)
    assert fpm.read_config(tmp_path / "c.json") == cfg


def test_dataset_round_trip(tmp_path):
    """write_dataset / read_dataset (io.cpp:321-384): frames/led_RR_CC.pgm,
    manifest "fpm-dataset/1", truth.cfi; frames, LEDs, timestamps and optics
    come back exactly."""
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=8, led_scan_rows=3, led_scan_cols=3)
    seq = fpm.led_sequence("spiral", cfg)
    rng = np.random.default_rng(8)
    imgs = rng.integers(0, 65536, (len(seq), 40, 48), dtype=np.uint16)
    fs = fpm.FrameSet(imgs, [tuple(l) for l in seq], np.arange(len(seq)) * 0.33)
    truth = rng.normal(size=(8, 8)) + 1j * rng.normal(size=(8, 8))
    fpm.write_dataset(tmp_path / "data", fs, cfg, object_truth=truth)
    assert (tmp_path / "data" / "frames" / "led_32_32.pgm").exists()
    ds = fpm.read_dataset(tmp_path / "data")
    assert np.array_equal(ds.frames.images, imgs)
    assert [tuple(l) for l in ds.frames.leds] == [tuple(l) for l in seq]
    assert np.array_equal(ds.frames.timestamps, fs.timestamps)
    assert ds.cfg == cfg
    assert np.array_equal(fpm.read_cfi(ds.object_truth), truth)


def test_dataset_manifest_checks(tmp_path):
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=8, led_scan_rows=3, led_scan_cols=3)
    fs = fpm.FrameSet(np.zeros((1, 8, 8), np.uint16), [(32, 32)], np.zeros(1))
    d = tmp_path / "d"
    fpm.write_dataset(d, fs, cfg)
    m = json.loads((d / "manifest.json").read_text())
    with pytest.raises(fpm.IoError, match="missing manifest.json"):
        fpm.read_dataset(tmp_path / "nothing")
    for mutate, exc, msg in [
        (lambda m: m.update(extra=1), fpm.ConfigError, 'unknown key "extra" in manifest'),
        (lambda m: m.update(format_version="fpm-dataset/2"), fpm.IoError, "unrecognized manifest version"),
        (lambda m: m["frames"][0].update(led_row=64), fpm.IoError, "manifest LED index outside grid"),
        (lambda m: m["frames"][0].update(file="frames/none.pgm"), fpm.IoError, "referenced frame missing"),
        (lambda m: m["frames"][0].pop("led_col"), fpm.IoError, "manifest frame entry missing required keys"),
    ]:
        mm = json.loads(json.dumps(m))
        mutate(mm)
        (d / "manifest.json").write_text(json.dumps(mm))
        with pytest.raises(exc, match=msg):
            fpm.read_dataset(d)
