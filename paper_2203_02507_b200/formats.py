"""Data formats on either side of the reconstruction path:
the reference's on-disk formats, so a reference user's datasets, configs and
outputs move through this engine unchanged (`include/fpm/io.hpp`,
`src/io.cpp`). The CLI itself is out of scope (tier framing); these are the
readers and writers it calls.

* PGM16 (`io.cpp:67-97`): "P5\\n<cols> <rows>\\n65535\\n", big-endian u16 samples.
* CFI (`io.cpp:99-137`): "CFI1", u32le width, u32le height, row-major (re, im)
  little-endian f64 pairs; non-finite values refused; round trips bit-exact.
* Views (`io.cpp:139-182`): amplitude ([0, max]) or phase ([-pi, pi]) to PGM16,
  the mapping in "<path>.meta.txt".
* Config JSON (`io.cpp:184-319`): {"optics": {...}, "run": {...}}, strict keys,
  defaults materialised on write.
* Dataset directory (`io.cpp:321-384`): frames/led_RR_CC.pgm + manifest.json
  ("fpm-dataset/1") + optional truth.cfi.

Error types and messages follow the reference (`IoError` for files,
`ConfigError` for config/manifest contents).
"""
from __future__ import annotations

import json
import math
import os
import struct
from dataclasses import dataclass, field

import numpy as np

from ._lib import ConfigError
from .engine import FrameSet, OpticalConfig


class IoError(RuntimeError):
    """io.hpp:12-14"""


# ------------------------------------------------------------------ PGM16
def write_pgm16(path, image) -> None:
    """io.cpp:67-74: header, then big-endian u16 samples row by row."""
    img = np.asarray(image)
    if img.ndim != 2:
        raise IoError("PGM image must be 2-D")
    rows, cols = img.shape
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{cols} {rows}\n65535\n".encode())
            f.write(np.ascontiguousarray(img, dtype=">u2").tobytes())
    except OSError:
        raise IoError(f"cannot open {os.fspath(path)} for writing") from None


def _tokens(buf: bytes, pos: int, count: int):
    """`is >> token` count times: whitespace-separated tokens (io.cpp:80-83)."""
    out = []
    n = len(buf)
    for _ in range(count):
        while pos < n and chr(buf[pos]).isspace():
            pos += 1
        start = pos
        while pos < n and not chr(buf[pos]).isspace():
            pos += 1
        out.append(buf[start:pos].decode("latin-1"))
    return out, pos


def read_pgm16(path) -> np.ndarray:
    """io.cpp:76-97; returns a [rows, cols] uint16 array."""
    p = os.fspath(path)
    try:
        with open(p, "rb") as f:
            buf = f.read()
    except OSError:
        raise IoError(f"cannot open {p}") from None
    (magic,), pos = _tokens(buf, 0, 1)
    if magic != "P5":
        raise IoError(f"not a binary PGM: {p}")
    toks, pos = _tokens(buf, pos, 3)
    try:
        w, h, maxval = (int(t) for t in toks)
    except ValueError:
        raise IoError(f"malformed PGM header: {p}") from None
    if w <= 0 or h <= 0:
        raise IoError(f"malformed PGM header: {p}")
    if maxval != 65535:
        raise IoError(f"PGM maxval must be 65535, got {maxval}")
    pos += 1  # single whitespace after maxval
    want = w * h * 2
    got = max(0, min(want, len(buf) - pos))
    if got != want:
        raise IoError(f"truncated PGM payload in {p}: expected {want} bytes, got {got}")
    return np.frombuffer(buf, dtype=">u2", count=w * h, offset=pos).astype(np.uint16).reshape(h, w)


# ------------------------------------------------------------------ CFI
def write_cfi(path, field_) -> None:
    """io.cpp:99-116: refuses non-finite values, naming the first pixel (row-major)."""
    f = np.asarray(field_, dtype=np.complex128)
    if f.ndim != 2:
        raise IoError("CFI field must be 2-D")
    bad = ~(np.isfinite(f.real) & np.isfinite(f.imag))
    if bad.any():
        i, j = np.argwhere(bad)[0]
        raise IoError(f"non-finite value at pixel ({i},{j})")
    rows, cols = f.shape
    try:
        with open(path, "wb") as fh:
            fh.write(b"CFI1")
            fh.write(struct.pack("<II", cols, rows))
            fh.write(np.ascontiguousarray(f, dtype="<c16").tobytes())
    except OSError:
        raise IoError(f"cannot open {os.fspath(path)} for writing") from None


def read_cfi(path) -> np.ndarray:
    """io.cpp:118-137; returns a [rows, cols] complex128 array (bit-exact)."""
    p = os.fspath(path)
    try:
        with open(p, "rb") as fh:
            buf = fh.read()
    except OSError:
        raise IoError(f"cannot open {p}") from None
    if len(buf) < 4 or buf[:4] != b"CFI1":
        raise IoError(f"bad CFI magic in {p}")
    if len(buf) < 12:
        raise IoError("unexpected end of file")
    w, h = struct.unpack_from("<II", buf, 4)
    if w == 0 or h == 0 or w * h > (1 << 30):
        raise IoError(f"CFI size out of range: {w}x{h}")
    if len(buf) < 12 + 16 * w * h:
        raise IoError("unexpected end of file")
    return np.frombuffer(buf, dtype="<c16", count=w * h, offset=12).astype(np.complex128).reshape(h, w)


# ------------------------------------------------------------------ views
def export_view(field_, which: str, path) -> None:
    """io.cpp:139-164: which = "amplitude" ([0, max], a zero field maps to zeros)
    or "phase" ([-pi, pi]); lround(t * 65535) clamped; sidecar "<path>.meta.txt"."""
    f = np.asarray(field_, dtype=np.complex128)
    if which == "amplitude":
        vals = np.abs(f)
        lo, hi = 0.0, float(vals.max()) if vals.size else 0.0
        if hi <= 0.0:
            hi = 1.0
    elif which == "phase":
        vals = np.angle(f)
        lo, hi = -math.pi, math.pi
    else:
        raise ConfigError(f"unknown view: {which}")
    t = (vals - lo) / (hi - lo) * 65535.0
    img = np.clip(np.where(t >= 0, np.floor(t + 0.5), np.ceil(t - 0.5)), 0, 65535).astype(np.uint16)  # lround
    write_pgm16(path, img)
    try:
        with open(os.fspath(path) + ".meta.txt", "w") as m:
            m.write(f"view {which}\nlo {lo:.17g}\nhi {hi:.17g}\n")
    except OSError:
        raise IoError(f"cannot write sidecar for {os.fspath(path)}") from None


def import_view(path) -> np.ndarray:
    """io.cpp:166-182: lo + (hi - lo) * v / 65535 per pixel."""
    p = os.fspath(path)
    try:
        with open(p + ".meta.txt") as m:
            toks = m.read().split()
    except OSError:
        raise IoError(f"missing sidecar for {p}") from None
    try:
        lo, hi = float(toks[3]), float(toks[5])
    except (IndexError, ValueError):
        raise IoError(f"malformed sidecar for {p}") from None
    img = read_pgm16(p)
    return lo + (hi - lo) * img.astype(np.float64) / 65535.0


# ------------------------------------------------------------------ config JSON
@dataclass
class NoiseSpec:
    enabled: bool = False
    photons: float = 1e4
    seed: int = 0


@dataclass
class RunConfig:
    """io.hpp:43-53"""
    iters: int = 5
    order: str = "spiral"
    workers: int = 1
    lag: int | None = None  # None = auto
    mode: str = "offline"
    online_delay: float = 1.0
    noise: NoiseSpec = field(default_factory=NoiseSpec)
    defocus_um: float = 0.0
    defocus_candidates_um: list = field(default_factory=list)


@dataclass
class AppConfig:
    optics: OpticalConfig = field(default_factory=OpticalConfig)
    run: RunConfig = field(default_factory=RunConfig)


_OPTICS_KEYS = ("wavelength_um", "objective_na", "magnification", "camera_pixel_um", "led_pitch_mm", "led_grid",
                "led_height_mm", "center_led", "led_scan", "upsample", "tile_size_px", "tile_overlap_px",
                "acq_pattern_delay_s", "acq_exposure_s")
_RUN_KEYS = ("iters", "order", "workers", "lag", "mode", "online_delay", "noise", "defocus_um",
             "defocus_candidates_um")


def _reject_unknown(j: dict, known, where: str) -> None:
    for k in j:
        if k not in known:
            raise ConfigError(f'unknown key "{k}" in {where}')


def optics_to_json(c: OpticalConfig) -> dict:
    """io.cpp:186-201"""
    return {"wavelength_um": c.wavelength, "objective_na": c.objective_na, "magnification": c.magnification,
            "camera_pixel_um": c.camera_pixel, "led_pitch_mm": c.led_pitch,
            "led_grid": [c.led_grid_rows, c.led_grid_cols], "led_height_mm": c.led_height,
            "center_led": [c.center_row, c.center_col], "led_scan": [c.led_scan_rows, c.led_scan_cols],
            "upsample": c.upsample, "tile_size_px": c.tile_size, "tile_overlap_px": c.tile_overlap,
            "acq_pattern_delay_s": c.acq_pattern_delay, "acq_exposure_s": c.acq_exposure}


def optics_from_json(j: dict) -> OpticalConfig:
    """io.cpp:203-235: defaults for absent keys, then OpticalConfig::validate."""
    if not isinstance(j, dict):
        raise ConfigError("config type error: optics must be an object")
    _reject_unknown(j, _OPTICS_KEYS, "optics")
    c = OpticalConfig()
    c.wavelength = float(j.get("wavelength_um", c.wavelength))
    c.objective_na = float(j.get("objective_na", c.objective_na))
    c.magnification = float(j.get("magnification", c.magnification))
    c.camera_pixel = float(j.get("camera_pixel_um", c.camera_pixel))
    c.led_pitch = float(j.get("led_pitch_mm", c.led_pitch))
    if "led_grid" in j:
        c.led_grid_rows, c.led_grid_cols = int(j["led_grid"][0]), int(j["led_grid"][1])
    c.led_height = float(j.get("led_height_mm", c.led_height))
    if "center_led" in j:
        c.center_row, c.center_col = int(j["center_led"][0]), int(j["center_led"][1])
    if "led_scan" in j:
        c.led_scan_rows, c.led_scan_cols = int(j["led_scan"][0]), int(j["led_scan"][1])
    c.upsample = int(j.get("upsample", c.upsample))
    c.tile_size = int(j.get("tile_size_px", c.tile_size))
    c.tile_overlap = int(j.get("tile_overlap_px", c.tile_overlap))
    c.acq_pattern_delay = float(j.get("acq_pattern_delay_s", c.acq_pattern_delay))
    c.acq_exposure = float(j.get("acq_exposure_s", c.acq_exposure))
    c.validate()
    return c


def run_to_json(r: RunConfig) -> dict:
    """io.cpp:237-249"""
    return {"iters": r.iters, "order": r.order, "workers": r.workers, "lag": "auto" if r.lag is None else r.lag,
            "mode": r.mode, "online_delay": r.online_delay,
            "noise": {"enabled": r.noise.enabled, "photons": r.noise.photons, "seed": r.noise.seed},
            "defocus_um": r.defocus_um, "defocus_candidates_um": list(r.defocus_candidates_um)}


def run_from_json(j: dict) -> RunConfig:
    """io.cpp:251-280"""
    if not isinstance(j, dict):
        raise ConfigError("config type error: run must be an object")
    _reject_unknown(j, _RUN_KEYS, "run")
    r = RunConfig()
    r.iters = int(j.get("iters", r.iters))
    r.order = str(j.get("order", r.order))
    r.workers = int(j.get("workers", r.workers))
    if "lag" in j and not isinstance(j["lag"], str):
        r.lag = int(j["lag"])
    r.mode = str(j.get("mode", r.mode))
    r.online_delay = float(j.get("online_delay", r.online_delay))
    if "noise" in j:
        n = j["noise"]
        _reject_unknown(n, ("enabled", "photons", "seed"), "run.noise")
        r.noise = NoiseSpec(bool(n.get("enabled", False)), float(n.get("photons", 1e4)), int(n.get("seed", 0)))
    r.defocus_um = float(j.get("defocus_um", 0.0))
    if "defocus_candidates_um" in j:
        r.defocus_candidates_um = [float(v) for v in j["defocus_candidates_um"]]
    if r.iters < 1:
        raise ConfigError("run.iters must be >= 1")
    if r.workers < 1:
        raise ConfigError("run.workers must be >= 1")
    if r.order not in ("spiral", "raster"):
        raise ConfigError("run.order must be spiral or raster")
    if r.mode not in ("offline", "online"):
        raise ConfigError("run.mode must be offline or online")
    return r


def config_to_json(cfg: AppConfig) -> str:
    """io.cpp:282-285: both sections with every default materialised (sorted keys,
    2-space indent, as nlohmann::json's dump(2))."""
    return json.dumps({"optics": optics_to_json(cfg.optics), "run": run_to_json(cfg.run)}, indent=2,
                      sort_keys=True) + "\n"


def config_from_json(text: str) -> AppConfig:
    """io.cpp:287-305"""
    try:
        j = json.loads(text)
    except ValueError as e:
        raise ConfigError(f"config parse error: {e}") from None
    if not isinstance(j, dict):
        raise ConfigError("config type error: top level must be an object")
    _reject_unknown(j, ("optics", "run"), "config")
    cfg = AppConfig()
    try:
        if "optics" in j:
            cfg.optics = optics_from_json(j["optics"])
        if "run" in j:
            cfg.run = run_from_json(j["run"])
    except (TypeError, IndexError, KeyError, ValueError) as e:
        raise ConfigError(f"config type error: {e}") from None
    return cfg


def read_config(path) -> AppConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise IoError(f"cannot open {os.fspath(path)}") from None
    return config_from_json(text)


def write_config(path, cfg: AppConfig) -> None:
    try:
        with open(path, "w") as f:
            f.write(config_to_json(cfg))
    except OSError:
        raise IoError(f"cannot open {os.fspath(path)} for writing") from None


# ------------------------------------------------------------------ dataset directory
@dataclass
class Dataset:
    """io.hpp:63-66 (the FrameSet's optics travel as `cfg`)."""
    frames: FrameSet
    cfg: OpticalConfig
    object_truth: str | None = None


def write_dataset(path, frames: FrameSet, cfg: OpticalConfig, object_truth=None) -> None:
    """io.cpp:321-345: frames/led_RR_CC.pgm per frame, manifest.json, truth.cfi."""
    d = os.fspath(path)
    os.makedirs(os.path.join(d, "frames"), exist_ok=True)
    flist = []
    ts = frames.timestamps if frames.timestamps is not None else np.zeros(len(frames.leds))
    for img, led, t in zip(frames.images, frames.leds, ts):
        name = f"frames/led_{int(led[0]):02d}_{int(led[1]):02d}.pgm"
        write_pgm16(os.path.join(d, name), img)
        flist.append({"file": name, "led_col": int(led[1]), "led_row": int(led[0]), "timestamp_s": float(t)})
    manifest = {"config": {"optics": optics_to_json(cfg)}, "format_version": "fpm-dataset/1", "frames": flist}
    if object_truth is not None:
        write_cfi(os.path.join(d, "truth.cfi"), object_truth)
        manifest["object_truth"] = "truth.cfi"
    try:
        with open(os.path.join(d, "manifest.json"), "w") as f:
            f.write(json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    except OSError:
        raise IoError(f"cannot write manifest in {d}") from None


def read_dataset(path) -> Dataset:
    """io.cpp:347-384. Frames must share one size (they are stacked [F, H, W])."""
    d = os.fspath(path)
    try:
        with open(os.path.join(d, "manifest.json")) as f:
            text = f.read()
    except OSError:
        raise IoError(f"missing manifest.json in {d}") from None
    try:
        manifest = json.loads(text)
    except ValueError as e:
        raise IoError(f"manifest parse error: {e}") from None
    _reject_unknown(manifest, ("format_version", "config", "frames", "object_truth"), "manifest")
    version = manifest.get("format_version", "")
    if version != "fpm-dataset/1":
        raise IoError(f"unrecognized manifest version: {version}")
    if "config" not in manifest or "frames" not in manifest:
        raise IoError("manifest missing required keys (config, frames)")
    cfg = optics_from_json(manifest["config"]["optics"])
    images, leds, ts = [], [], []
    for fj in manifest["frames"]:
        if not all(k in fj for k in ("file", "led_row", "led_col")):
            raise IoError("manifest frame entry missing required keys")
        row, col = int(fj["led_row"]), int(fj["led_col"])
        if row < 0 or row >= cfg.led_grid_rows or col < 0 or col >= cfg.led_grid_cols:
            raise IoError("manifest LED index outside grid")
        file = os.path.join(d, fj["file"])
        if not os.path.exists(file):
            raise IoError(f"referenced frame missing: {file}")
        images.append(read_pgm16(file))
        leds.append((row, col))
        ts.append(float(fj.get("timestamp_s", 0.0)))
    if images and any(im.shape != images[0].shape for im in images):
        raise IoError("dataset frames differ in size")
    truth = None
    if "object_truth" in manifest:
        truth = os.path.join(d, manifest["object_truth"])
        if not os.path.exists(truth):
            raise IoError(f"referenced truth missing: {truth}")
    stack = np.stack(images) if images else np.zeros((0, 0, 0), np.uint16)
    return Dataset(FrameSet(stack, leds, np.asarray(ts)), cfg, truth)
