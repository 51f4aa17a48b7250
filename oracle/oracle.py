"""ctypes view of the CPU oracle (oracle/lib/libfpm_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, as the checker and the CPU
baseline. The product package never imports this module.

The oracle restates the reference (/root/reference/proj, C++/Eigen) in plain
C++ double; see fpm_oracle.hpp for the file:line map. Complex arrays cross the
boundary as numpy complex128, row-major.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field, fields

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libfpm_oracle.so")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str, minimum: int | None = None):
        super().__init__(msg)
        self.code = code
        self.minimum = minimum


class ConfigError(OracleError):
    pass


class DataError(OracleError):
    pass


class UnsafeLagError(OracleError):
    pass


class DomainError(OracleError):
    pass


_ERRS = {1: ConfigError, 2: DataError, 3: UnsafeLagError, 4: DomainError}


class OrcConfig(C.Structure):
    _fields_ = [
        ("wavelength", C.c_double), ("objective_na", C.c_double), ("magnification", C.c_double),
        ("camera_pixel", C.c_double), ("led_pitch", C.c_double),
        ("led_grid_rows", C.c_int), ("led_grid_cols", C.c_int),
        ("led_height", C.c_double),
        ("center_row", C.c_int), ("center_col", C.c_int), ("led_scan_rows", C.c_int),
        ("led_scan_cols", C.c_int), ("upsample", C.c_int), ("tile_size", C.c_int),
        ("tile_overlap", C.c_int),
        ("acq_pattern_delay", C.c_double), ("acq_exposure", C.c_double),
    ]


@dataclass
class Optics:
    """OpticalConfig with the reference defaults (optics.hpp:29-52)."""
    wavelength: float = 0.525
    objective_na: float = 0.1
    magnification: float = 2.0
    camera_pixel: float = 2.4
    led_pitch: float = 2.5
    led_grid_rows: int = 64
    led_grid_cols: int = 64
    led_height: float = 83.0
    center_row: int = 32
    center_col: int = 32
    led_scan_rows: int = 13
    led_scan_cols: int = 13
    upsample: int = 4
    tile_size: int = 256
    tile_overlap: int = 26
    acq_pattern_delay: float = 0.3
    acq_exposure: float = 0.03

    def c(self) -> OrcConfig:
        return OrcConfig(**{f.name: getattr(self, f.name) for f in fields(self)})

    @property
    def hr_size(self) -> int:
        return self.tile_size * self.upsample

    @property
    def dx_obj(self) -> float:
        return self.camera_pixel / self.magnification

    @property
    def center_led(self):
        return (self.center_row, self.center_col)


def toy_cfg(**kw) -> Optics:
    """test_util.hpp:11-19: tile 64, overlap 8, upsample 4, 3x3 scan."""
    base = dict(tile_size=64, tile_overlap=8, upsample=4, led_scan_rows=3, led_scan_cols=3)
    base.update(kw)
    return Optics(**base)


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
    return _lib


def _call(name: str, *args) -> None:
    L = lib()
    rc = getattr(L, name)(*args)
    if rc != 0:
        msg = L.orc_last_error().decode()
        cls = _ERRS.get(rc, OracleError)
        raise cls(rc, msg, L.orc_last_min_lag() if rc == 3 else None)


def _p(a: np.ndarray, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


def _cplx(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _seq_arr(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int32).reshape(-1, 2))


# ------------------------------------------------------------------ field
def fft2(x, threads: int = 1) -> np.ndarray:
    x = _cplx(x)
    out = np.empty_like(x)
    _call("orc_fft2", _p(x), x.shape[0], x.shape[1], 0, threads, _p(out))
    return out


def ifft2(x, threads: int = 1) -> np.ndarray:
    x = _cplx(x)
    out = np.empty_like(x)
    _call("orc_fft2", _p(x), x.shape[0], x.shape[1], 1, threads, _p(out))
    return out


def fftshift(x, inverse: bool = False) -> np.ndarray:
    x = _cplx(x)
    out = np.empty_like(x)
    _call("orc_fftshift", _p(x), x.shape[0], x.shape[1], int(inverse), _p(out))
    return out


def upsample_bilinear(x, factor: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty((x.shape[0] * factor, x.shape[1] * factor))
    _call("orc_upsample_bilinear", _p(x), x.shape[0], x.shape[1], factor, _p(out))
    return out


# ------------------------------------------------------------------ optics / tiles
def validate(cfg: Optics) -> None:
    c = cfg.c()
    _call("orc_validate", C.byref(c))


def illumination_wavevector(led, center_um, cfg: Optics):
    fx, fy = C.c_double(), C.c_double()
    c = cfg.c()
    _call("orc_illumination_wavevector", C.byref(c), int(led[0]), int(led[1]),
          C.c_double(center_um[0]), C.c_double(center_um[1]), C.byref(fx), C.byref(fy))
    return fx.value, fy.value


def build_pupil(cfg: Optics, grid: int, defocus_um: float = 0.0):
    vals = np.zeros((max(grid, 1), max(grid, 1)), np.complex128)
    r = C.c_double()
    c = cfg.c()
    _call("orc_build_pupil", C.byref(c), grid, C.c_double(defocus_um), _p(vals), C.byref(r))
    return vals, r.value


def synthesized_na(cfg: Optics) -> float:
    out = C.c_double()
    c = cfg.c()
    _call("orc_synthesized_na", C.byref(c), C.byref(out))
    return out.value


def tile_origins(fov: int, tile: int, overlap: int):
    buf = np.zeros(4096, np.int32)
    n = C.c_int()
    _call("orc_tile_origins", fov, tile, overlap, _p(buf, C.c_int), 4096, C.byref(n))
    return buf[: n.value].tolist()


@dataclass
class Tiles:
    xy: np.ndarray       # [T, 2] (x0, y0)
    center: np.ndarray   # [T, 2] um
    kvecs: np.ndarray    # [T, L, 2] (fx, fy)
    offsets: np.ndarray  # [T, L, 2] (oy, ox)


def partition_tiles(fov_w: int, fov_h: int, cfg: Optics, seq) -> Tiles:
    s = _seq_arr(seq)
    L = len(s)
    nx = len(tile_origins(fov_w, cfg.tile_size, cfg.tile_overlap))
    ny = len(tile_origins(fov_h, cfg.tile_size, cfg.tile_overlap))
    T = nx * ny
    xy = np.zeros((T, 2), np.int32)
    ce = np.zeros((T, 2))
    kv = np.zeros((T, L, 2))
    of = np.zeros((T, L, 2), np.int32)
    n = C.c_int()
    c = cfg.c()
    _call("orc_partition_tiles", C.byref(c), fov_w, fov_h, _p(s, C.c_int), L, T, C.byref(n),
          _p(xy, C.c_int), _p(ce), _p(kv), _p(of, C.c_int))
    assert n.value == T
    return Tiles(xy, ce, kv, of)


def sequence_offsets(order: str, rows: int, cols: int):
    out = np.zeros((max(rows * cols, 1), 2), np.int32)
    _call("orc_sequence_offsets", 1 if order == "raster" else 0, rows, cols, _p(out, C.c_int))
    return [tuple(x) for x in out.tolist()]


def led_sequence(order: str, cfg: Optics):
    return [(cfg.center_row + r, cfg.center_col + c)
            for r, c in sequence_offsets(order, cfg.led_scan_rows, cfg.led_scan_cols)]


def spectrum_offset_px(kvec, cfg: Optics):
    oy, ox = C.c_int(), C.c_int()
    c = cfg.c()
    _call("orc_spectrum_offset_px", C.byref(c), C.c_double(kvec[0]), C.c_double(kvec[1]),
          C.byref(oy), C.byref(ox))
    return oy.value, ox.value


def min_safe_lag(offsets, radius: float) -> int:
    o = _seq_arr(offsets)
    out = C.c_int()
    _call("orc_min_safe_lag", _p(o, C.c_int), len(o), C.c_double(radius), C.byref(out))
    return out.value


def min_safe_lag_tile(cfg: Optics, fov_w: int, fov_h: int, tile_index: int, seq) -> int:
    s = _seq_arr(seq)
    out = C.c_int()
    c = cfg.c()
    _call("orc_min_safe_lag_tile", C.byref(c), fov_w, fov_h, tile_index, _p(s, C.c_int), len(s),
          C.byref(out))
    return out.value


def build_schedule(positions: int, iters: int, lag: int):
    ent = np.zeros((max(positions * iters, 1), 3), np.int32)
    rounds = C.c_int()
    _call("orc_build_schedule", positions, iters, lag, _p(ent, C.c_int), C.byref(rounds))
    return rounds.value, ent


# ------------------------------------------------------------------ forward
KINDS = {"bars": 0, "phase-disk": 1, "composite": 2}


def synth_object(kind: str, size: int, seed: int) -> np.ndarray:
    out = np.zeros((size, size), np.complex128)
    _call("orc_synth_object", KINDS[kind], size, C.c_ulonglong(seed), _p(out))
    return out


@dataclass
class FrameStack:
    """Frames [F, H, W] u16 row-major with their LED identities (forward.hpp:12-26)."""
    images: np.ndarray
    leds: list
    timestamps: np.ndarray = field(default_factory=lambda: np.zeros(0))

    @property
    def height(self) -> int:
        return self.images.shape[1]

    @property
    def width(self) -> int:
        return self.images.shape[2]

    def find(self, led):
        for i, l in enumerate(self.leds):
            if tuple(l) == tuple(led):
                return i
        return None


def simulate_dataset(obj, seq, cfg: Optics, noise: tuple | None = None,
                     defocus_um: float = 0.0) -> FrameStack:
    obj = _cplx(obj)
    s = _seq_arr(seq)
    L = len(s)
    H, W = obj.shape[0] // cfg.upsample, obj.shape[1] // cfg.upsample
    frames = np.zeros((L, H, W), np.uint16)
    ts = np.zeros(L)
    en, photons, nseed = (0, 1e4, 0) if noise is None else (1, noise[0], noise[1])
    c = cfg.c()
    _call("orc_simulate_dataset", _p(obj), obj.shape[0], obj.shape[1], C.byref(c), _p(s, C.c_int), L,
          en, C.c_double(photons), C.c_ulonglong(nseed), C.c_double(defocus_um),
          _p(frames, C.c_uint16), _p(ts))
    return FrameStack(frames, [tuple(x) for x in s.tolist()], ts)


def simulate_intensity(obj, kvec, cfg: Optics, defocus_um: float = 0.0) -> np.ndarray:
    obj = _cplx(obj)
    out = np.zeros((cfg.tile_size, cfg.tile_size))
    c = cfg.c()
    _call("orc_simulate_intensity", _p(obj), C.byref(c), C.c_double(kvec[0]), C.c_double(kvec[1]),
          C.c_double(defocus_um), _p(out))
    return out


# ------------------------------------------------------------------ recon
def _frames_args(fs: FrameStack):
    imgs = np.ascontiguousarray(fs.images, dtype=np.uint16)
    leds = _seq_arr(fs.leds)
    return imgs, leds


def init_canvas(fs: FrameStack, cfg: Optics, tile_index: int = 0) -> np.ndarray:
    imgs, leds = _frames_args(fs)
    out = np.zeros((cfg.hr_size, cfg.hr_size), np.complex128)
    c = cfg.c()
    _call("orc_init_canvas", C.byref(c), _p(imgs, C.c_uint16), _p(leds, C.c_int), len(leds),
          fs.height, fs.width, tile_index, _p(out))
    return out


def canvas_to_field(canvas, cfg: Optics) -> np.ndarray:
    canvas = _cplx(canvas)
    out = np.empty_like(canvas)
    c = cfg.c()
    _call("orc_canvas_to_field", C.byref(c), _p(canvas), _p(out))
    return out


def update_step(canvas: np.ndarray, intensity, kvec, pupil, cfg: Optics) -> float:
    """In-place GS step on `canvas` (complex128 C-contiguous)."""
    assert canvas.dtype == np.complex128 and canvas.flags.c_contiguous
    I = np.ascontiguousarray(intensity, dtype=np.float64)
    P = _cplx(pupil)
    r = C.c_double()
    c = cfg.c()
    _call("orc_update_step", C.byref(c), _p(canvas), _p(I), C.c_double(kvec[0]), C.c_double(kvec[1]),
          _p(P), C.byref(r))
    return r.value


def update_step_epry(canvas: np.ndarray, intensity, kvec, pupil: np.ndarray, cfg: Optics,
                     alpha: float = 1.0, beta: float = 1.0, support=None) -> float:
    assert canvas.dtype == np.complex128 and canvas.flags.c_contiguous
    assert pupil.dtype == np.complex128 and pupil.flags.c_contiguous
    I = np.ascontiguousarray(intensity, dtype=np.float64)
    S = None if support is None else np.ascontiguousarray(support, dtype=np.uint8)
    r = C.c_double()
    c = cfg.c()
    _call("orc_update_step_epry", C.byref(c), _p(canvas), _p(I), C.c_double(kvec[0]),
          C.c_double(kvec[1]), _p(pupil), None if S is None else _p(S, C.c_uint8),
          C.c_double(alpha), C.c_double(beta), C.byref(r))
    return r.value


@dataclass
class TileResult:
    hr: np.ndarray
    residuals: np.ndarray
    pupil: np.ndarray
    lag: int = 1
    nondeterministic: bool = False
    wall_s: float = 0.0


MODES = {"gs": 0, "epry": 1}


def reconstruct_tile(fs: FrameStack, cfg: Optics, iters: int, seq, tile_index: int = 0,
                     mode: str = "gs", alpha: float = 1.0, beta: float = 1.0,
                     tile_defocus: float = 0.0, fft_threads: int = 1, pipelined: bool = False,
                     lag: int | None = None, force_unsafe: bool = False) -> TileResult:
    imgs, leds = _frames_args(fs)
    s = _seq_arr(seq)
    N, n = cfg.hr_size, cfg.tile_size
    hr = np.zeros((N, N), np.complex128)
    res = np.zeros(max(iters, 1))
    pup = np.zeros((n, n), np.complex128)
    lag_out, nd, wall = C.c_int(), C.c_int(), C.c_double()
    c = cfg.c()
    _call("orc_reconstruct_tile", C.byref(c), _p(imgs, C.c_uint16), _p(leds, C.c_int), len(leds),
          fs.height, fs.width, tile_index, C.c_double(tile_defocus), iters, _p(s, C.c_int), len(s),
          MODES[mode], C.c_double(alpha), C.c_double(beta), fft_threads, int(pipelined),
          -1 if lag is None else int(lag), int(force_unsafe), _p(hr), _p(res), _p(pup),
          C.byref(lag_out), C.byref(nd), C.byref(wall))
    return TileResult(hr, res[:iters], pup, lag_out.value, bool(nd.value), wall.value)


@dataclass
class OfflineResult:
    tiles: np.ndarray | None
    stitched: np.ndarray | None
    residuals: np.ndarray
    tile_count: int
    wall_s: float


def run_offline(fs: FrameStack, cfg: Optics, seq, iters: int, workers: int = 1,
                lag: int | None = None, force_unsafe: bool = False, force_pipeline: bool = False,
                defocus_um: float = 0.0, max_tiles: int | None = None, tile_defocus=None,
                mode: str = "gs", alpha: float = 1.0, beta: float = 1.0,
                want_tiles: bool = True, want_stitched: bool = True) -> OfflineResult:
    imgs, leds = _frames_args(fs)
    s = _seq_arr(seq)
    nx = len(tile_origins(fs.width, cfg.tile_size, cfg.tile_overlap))
    ny = len(tile_origins(fs.height, cfg.tile_size, cfg.tile_overlap))
    T = nx * ny if max_tiles is None else max_tiles
    N = cfg.hr_size
    tiles = np.zeros((T, N, N), np.complex128) if want_tiles else None
    st = (np.zeros((fs.height * cfg.upsample, fs.width * cfg.upsample), np.complex128)
          if (want_stitched and max_tiles is None) else None)
    resid = np.zeros((T, iters))
    td = None if tile_defocus is None else np.ascontiguousarray(tile_defocus, dtype=np.float64)
    cnt, wall = C.c_int(), C.c_double()
    c = cfg.c()
    _call("orc_run_offline", C.byref(c), _p(imgs, C.c_uint16), _p(leds, C.c_int), len(leds),
          fs.height, fs.width, _p(s, C.c_int), len(s), iters, workers, -1 if lag is None else lag,
          int(force_unsafe), int(force_pipeline), C.c_double(defocus_um),
          -1 if max_tiles is None else max_tiles, None if td is None else _p(td),
          0 if td is None else len(td), MODES[mode], C.c_double(alpha), C.c_double(beta),
          None if tiles is None else _p(tiles), None if st is None else _p(st), _p(resid),
          C.byref(cnt), C.byref(wall))
    return OfflineResult(tiles, st, resid, cnt.value, wall.value)


# ------------------------------------------------------------------ stitch / metrics
def mean_ratio(f1, f2, overlap: int, vertical: bool = False) -> complex:
    a, b = _cplx(f1), _cplx(f2)
    out = np.zeros(2)
    _call("orc_mean_ratio", _p(a), *a.shape, _p(b), *b.shape, overlap, int(vertical), _p(out))
    return complex(out[0], out[1])


def stitch_pair(f1, f2, overlap: int, vertical: bool = False) -> np.ndarray:
    a, b = _cplx(f1), _cplx(f2)
    r, c = C.c_int(), C.c_int()
    _call("orc_stitch_pair", _p(a), *a.shape, _p(b), *b.shape, overlap, int(vertical), None,
          C.byref(r), C.byref(c))
    out = np.zeros((r.value, c.value), np.complex128)
    _call("orc_stitch_pair", _p(a), *a.shape, _p(b), *b.shape, overlap, int(vertical), _p(out),
          C.byref(r), C.byref(c))
    return out


def stitch_mosaic(tiles, xy, cfg: Optics) -> np.ndarray:
    t = _cplx(tiles)
    xy = np.ascontiguousarray(xy, dtype=np.int32)
    r, c = C.c_int(), C.c_int()
    cc = cfg.c()
    _call("orc_stitch_mosaic", C.byref(cc), _p(t), _p(xy, C.c_int), len(xy), None, C.byref(r), C.byref(c))
    out = np.zeros((r.value, c.value), np.complex128)
    _call("orc_stitch_mosaic", C.byref(cc), _p(t), _p(xy, C.c_int), len(xy), _p(out), C.byref(r), C.byref(c))
    return out


def band_limit(field_, na: float, cfg: Optics) -> np.ndarray:
    f = _cplx(field_)
    out = np.empty_like(f)
    c = cfg.c()
    _call("orc_band_limit", _p(f), f.shape[0], C.c_double(na), C.byref(c), _p(out))
    return out


def global_alignment(recon, truth) -> complex:
    a, b = _cplx(recon), _cplx(truth)
    out = np.zeros(2)
    _call("orc_global_alignment", _p(a), _p(b), a.shape[0], a.shape[1], _p(out))
    return complex(out[0], out[1])


def rmse(a, b):
    """(amplitude_rmse, phase_rmse) (metrics.cpp:35-57)."""
    a, b = _cplx(a), _cplx(b)
    amp, ph = C.c_double(), C.c_double()
    _call("orc_rmse", _p(a), _p(b), a.shape[0], a.shape[1], C.byref(amp), C.byref(ph))
    return amp.value, ph.value
