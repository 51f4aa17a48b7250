"""Host-side mirror of the reference's reconstruct API over the C-ABI.

Names, argument meaning and errors follow /root/reference/proj:
  OpticalConfig / WaveVector / Pupil      include/fpm/optics.hpp:29-67
  TileSpec, tile_origins, partition_tiles include/fpm/tiles.hpp:13-28
  sequence_offsets, led_sequence, spectrum_offset_px, init_canvas,
  canvas_to_field, update_step, reconstruct_tile   include/fpm/recon.hpp:17-71
  min_safe_lag, build_schedule, pipelined_reconstruct_tile, run_offline
                                          include/fpm/parallel.hpp:19-91
All arithmetic runs in libfpm_b200.so: geometry in host C++ double (exact
reference formulas), every transform and update on the B200.
"""
from __future__ import annotations

import ctypes as C
import sys
import time
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib
from ._lib import (MODE_EPRY, MODE_GS, ORDER_RASTER, ORDER_SPIRAL, ConfigError, DataError,  # noqa: F401
                   DomainError, UnsafeLagError, check, lib)

MODES = {"gs": MODE_GS, "epry": MODE_EPRY}


@dataclass
class OpticalConfig:
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

    def c(self) -> _lib.OpticalConfigC:
        return _lib.OpticalConfigC(**{f.name: getattr(self, f.name) for f in fields(self)})

    @property
    def center_led(self):
        return (self.center_row, self.center_col)

    def dx_obj(self) -> float:
        return self.camera_pixel / self.magnification

    def dx_hr(self) -> float:
        return self.dx_obj() / self.upsample

    def hr_size(self) -> int:
        return self.tile_size * self.upsample

    def validate(self) -> None:
        c = self.c()
        check(lib().fpmgpu_validate_config(C.byref(c)))


@dataclass
class Pupil:
    grid: int
    radius_px: float
    defocus: float
    values: np.ndarray  # complex128 [grid, grid]


@dataclass
class TileSpec:
    x0: int = 0
    y0: int = 0
    size: int = 0
    center_x_um: float = 0.0
    center_y_um: float = 0.0
    defocus_um: float = 0.0
    wavevectors: dict = field(default_factory=dict)  # (row, col) -> (fx, fy)


@dataclass
class FrameSet:
    """LR intensity stack (forward.hpp:12-26): images [F, H, W] u16 with LED ids."""
    images: np.ndarray
    leds: list
    timestamps: np.ndarray | None = None

    def find(self, led):
        led = tuple(led)
        for i, l in enumerate(self.leds):
            if tuple(l) == led:
                return i
        return None

    def width(self) -> int:
        return int(self.images.shape[2])

    def height(self) -> int:
        return int(self.images.shape[1])


@dataclass
class SpectrumCanvas:
    spectrum: np.ndarray  # complex64 [N, N]
    cfg: OpticalConfig
    updated_offsets: list = field(default_factory=list)

    def size(self) -> int:
        return int(self.spectrum.shape[0])


@dataclass
class ReconMetrics:
    pass_mean_residual: list = field(default_factory=list)
    wall_s: float = 0.0


@dataclass
class ReconResult:
    hr: np.ndarray
    metrics: ReconMetrics
    pupil: np.ndarray | None = None


@dataclass
class PipelineResult:
    hr: np.ndarray
    metrics: ReconMetrics
    lag: int = 1
    nondeterministic: bool = False


@dataclass
class PipelineSchedule:
    lag: int
    stages: int
    rounds: list


@dataclass
class RunOptions:
    """parallel.hpp:79-87 plus the GPU extensions used by BASELINE configs 3-5."""
    iters: int = 5
    workers: int = 1
    lag: int | None = None
    force_unsafe_lag: bool = False
    force_pipeline: bool = False
    defocus_um: float = 0.0
    max_tiles: int | None = None
    tile_defocus_um: list | None = None
    mode: str = "gs"
    alpha: float = 1.0
    beta: float = 1.0


@dataclass
class TimingRow:
    run_id: str = ""
    mode: str = "offline"
    workers: int = 1
    lag: int = 1
    tiles: int = 1
    iters: int = 1
    wall_s: float = 0.0
    per_tile_mean_s: float = 0.0


@dataclass
class RunResult:
    specs: list
    tiles: np.ndarray  # complex64 [T, N, N]
    stitched: np.ndarray | None
    timing: TimingRow
    tile_metrics: list
    pupils: np.ndarray | None = None
    acquisition_s: float = 0.0  # online mode only (parallel.hpp:76)


def _p(a, ctype=C.c_int):
    return a.ctypes.data_as(C.POINTER(ctype))


# ------------------------------------------------------------------ geometry
def illumination_wavevector(led, tile_center_um, cfg: OpticalConfig):
    fx, fy = C.c_double(), C.c_double()
    c = cfg.c()
    check(lib().fpmgpu_illumination_wavevector(C.byref(c), int(led[0]), int(led[1]),
                                               C.c_double(tile_center_um[0]), C.c_double(tile_center_um[1]),
                                               C.byref(fx), C.byref(fy)))
    return fx.value, fy.value


def build_pupil(cfg: OpticalConfig, grid: int, defocus_um: float = 0.0) -> Pupil:
    vals = np.zeros((max(grid, 1), max(grid, 1)), np.complex128)
    r = C.c_double()
    c = cfg.c()
    check(lib().fpmgpu_build_pupil(C.byref(c), int(grid), C.c_double(defocus_um),
                                   vals.ctypes.data_as(C.POINTER(C.c_double)), C.byref(r)))
    return Pupil(grid, r.value, defocus_um, vals)


def synthesized_na(cfg: OpticalConfig) -> float:
    out = C.c_double()
    c = cfg.c()
    check(lib().fpmgpu_synthesized_na(C.byref(c), C.byref(out)))
    return out.value


def tile_origins(fov: int, tile_size: int, tile_overlap: int) -> list:
    cap = max(1, fov + 2)
    buf = np.zeros(cap, np.int32)
    n = C.c_int()
    check(lib().fpmgpu_tile_origins(int(fov), int(tile_size), int(tile_overlap), _p(buf), cap, C.byref(n)))
    return buf[: n.value].tolist()


def sequence_offsets(order: str, rows: int, cols: int) -> list:
    if order not in ("spiral", "raster"):
        raise ConfigError(f"unknown update order: {order}")
    out = np.zeros((max(rows * cols, 1), 2), np.int32)
    check(lib().fpmgpu_sequence_offsets(ORDER_RASTER if order == "raster" else ORDER_SPIRAL, rows, cols, _p(out)))
    return [tuple(x) for x in out[: rows * cols].tolist()]


def led_sequence(order: str, cfg: OpticalConfig) -> list:
    return [(cfg.center_row + r, cfg.center_col + c)
            for r, c in sequence_offsets(order, cfg.led_scan_rows, cfg.led_scan_cols)]


def scan_leds(cfg: OpticalConfig) -> list:
    hr, hc = cfg.led_scan_rows // 2, cfg.led_scan_cols // 2
    return [(cfg.center_row + dr, cfg.center_col + dc) for dr in range(-hr, hr + 1) for dc in range(-hc, hc + 1)]


def partition_arrays(fov_w: int, fov_h: int, cfg: OpticalConfig, leds):
    """Vectorised partition_tiles: xy [T,2], centers [T,2], kvecs [T,L,2], offsets [T,L,2]."""
    s = np.ascontiguousarray(np.asarray(leds, np.int32).reshape(-1, 2))
    L = len(s)
    T = len(tile_origins(fov_w, cfg.tile_size, cfg.tile_overlap)) * len(
        tile_origins(fov_h, cfg.tile_size, cfg.tile_overlap))
    xy = np.zeros((T, 2), np.int32)
    ce = np.zeros((T, 2))
    kv = np.zeros((T, L, 2))
    of = np.zeros((T, L, 2), np.int32)
    n = C.c_int()
    c = cfg.c()
    check(lib().fpmgpu_partition_tiles(C.byref(c), int(fov_w), int(fov_h), _p(s), L, T, C.byref(n), _p(xy),
                                       _p(ce, C.c_double), _p(kv, C.c_double), _p(of)))
    return xy, ce, kv, of


def partition_tiles(fov_w: int, fov_h: int, cfg: OpticalConfig, defocus_um: float = 0.0) -> list:
    leds = scan_leds(cfg)
    xy, ce, kv, _ = partition_arrays(fov_w, fov_h, cfg, leds)
    out = []
    for t in range(len(xy)):
        out.append(TileSpec(int(xy[t, 0]), int(xy[t, 1]), cfg.tile_size, float(ce[t, 0]), float(ce[t, 1]),
                            defocus_um, {led: (float(kv[t, k, 0]), float(kv[t, k, 1])) for k, led in enumerate(leds)}))
    return out


def spectrum_offset_px(wv, cfg: OpticalConfig):
    oy, ox = C.c_int(), C.c_int()
    c = cfg.c()
    check(lib().fpmgpu_spectrum_offset_px(C.byref(c), C.c_double(wv[0]), C.c_double(wv[1]), C.byref(oy),
                                          C.byref(ox)))
    return oy.value, ox.value


def min_safe_lag(offsets_px, radius_px: float) -> int:
    o = np.ascontiguousarray(np.asarray(offsets_px, np.int32).reshape(-1, 2))
    out = C.c_int()
    check(lib().fpmgpu_min_safe_lag(_p(o), len(o), C.c_double(radius_px), C.byref(out)))
    return out.value


def min_safe_lag_tile(seq, tile: TileSpec, cfg: OpticalConfig) -> int:
    offs = [spectrum_offset_px(tile.wavevectors[tuple(l)], cfg) for l in seq]
    return min_safe_lag(offs, build_pupil(cfg, cfg.tile_size, tile.defocus_um).radius_px)


def build_schedule(positions: int, iters: int, lag: int) -> PipelineSchedule:
    ent = np.zeros((max(positions * iters, 1), 3), np.int32)
    rounds = C.c_int()
    check(lib().fpmgpu_build_schedule(int(positions), int(iters), int(lag), _p(ent), C.byref(rounds)))
    rr = [[] for _ in range(rounds.value)]
    for r, s, p in ent[: positions * iters].tolist():
        rr[r].append((s, p))
    return PipelineSchedule(lag, iters, rr)


# ------------------------------------------------------------------ engine
class Engine:
    """A device context (fpmgpu_context) on one GPU."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().fpmgpu_create(int(device), C.byref(self._h)))
        self.device = device

    def close(self):
        if self._h:
            lib().fpmgpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h


_engines: dict = {}


def default_engine(device: int = 0) -> Engine:
    if device not in _engines:
        _engines[device] = Engine(device)
    return _engines[device]


@dataclass
class Request:
    """Geometry of one batched reconstruction (fpmgpu_recon_request)."""
    cfg: OpticalConfig
    iters: int
    tile_xy: np.ndarray       # [T, 2] int32
    offsets: np.ndarray       # [T, L, 2] int32
    seq_frame: np.ndarray     # [L] int32
    init_frame: int
    num_frames: int
    height: int
    width: int
    mode: str = "gs"
    alpha: float = 1.0
    beta: float = 1.0
    lag: int = 0
    force_unsafe_lag: bool = False
    tile_defocus_um: np.ndarray | None = None
    pupils: np.ndarray | None = None  # complex64 [T, n, n]

    def c(self):
        keep = []
        xy = np.ascontiguousarray(self.tile_xy, np.int32)
        of = np.ascontiguousarray(self.offsets, np.int32)
        sf = np.ascontiguousarray(self.seq_frame, np.int32)
        keep += [xy, of, sf]
        r = _lib.ReconRequestC()
        r.cfg = self.cfg.c()
        r.iters = self.iters
        r.mode = MODES[self.mode]
        r.alpha, r.beta = self.alpha, self.beta
        r.lag = self.lag
        r.force_unsafe_lag = int(self.force_unsafe_lag)
        r.num_tiles = len(xy)
        r.tile_xy = _p(xy)
        r.num_leds = len(sf)
        r.offsets = _p(of)
        r.seq_frame = _p(sf)
        r.init_frame = int(self.init_frame)
        if self.tile_defocus_um is not None:
            td = np.ascontiguousarray(self.tile_defocus_um, np.float64)
            keep.append(td)
            r.tile_defocus_um = _p(td, C.c_double)
        if self.pupils is not None:
            pu = np.ascontiguousarray(self.pupils, np.complex64)
            keep.append(pu)
            r.pupils = pu.ctypes.data_as(C.POINTER(C.c_float))
        r.num_frames, r.height, r.width = self.num_frames, self.height, self.width
        return r, keep


def make_request(frames: FrameSet, cfg: OpticalConfig, seq, tiles: list, iters: int, **kw) -> Request:
    """Resolve LEDs to frames (recon.cpp:146-156), offsets (recon.cpp:50-53) and the
    init seed (recon.cpp:62-75) for a list of TileSpecs."""
    if iters < 1:
        raise ConfigError("iters must be >= 1")
    seq_frame = []
    for led in seq:
        f = frames.find(led)
        if f is None:
            raise DataError(f"missing frame for LED ({led[0]},{led[1]})")
        seq_frame.append(f)
    init = frames.find(cfg.center_led)
    if init is None:
        print("fpm: warning: on-axis frame missing, initializing from brightest frame", file=sys.stderr)
        if len(frames.leds) == 0:
            raise DataError("empty frame set")
        init = int(np.argmax(frames.images.reshape(len(frames.leds), -1).mean(axis=1)))
    T, L = len(tiles), len(seq)
    xy = np.array([[t.x0, t.y0] for t in tiles], np.int32).reshape(T, 2)
    of = np.zeros((T, L, 2), np.int32)
    for i, t in enumerate(tiles):
        for k, led in enumerate(seq):
            of[i, k] = spectrum_offset_px(t.wavevectors[tuple(led)], cfg)
    defocus = np.array([t.defocus_um for t in tiles], np.float64)
    return Request(cfg, iters, xy, of, np.array(seq_frame, np.int32), init, len(frames.leds),
                   frames.height(), frames.width(), tile_defocus_um=defocus if np.any(defocus) else None, **kw)


def reconstruct_request(req: Request, frames: FrameSet, engine: Engine | None = None):
    """fpmgpu_reconstruct_tiles on host buffers -> (hr [T,N,N] c64, residuals [T,iters], pupils, lag)."""
    eng = engine or default_engine()
    r, keep = req.c()
    T, n, N = r.num_tiles, req.cfg.tile_size, req.cfg.hr_size()
    imgs = np.ascontiguousarray(frames.images, np.uint16)
    hr = np.zeros((T, N, N), np.complex64)
    res = np.zeros((T, req.iters), np.float64)
    pup = np.zeros((T, n, n), np.complex64)
    lag = C.c_int()
    check(lib().fpmgpu_reconstruct_tiles(eng.handle, C.byref(r), imgs.ctypes.data, imgs.shape[2],
                                         hr.ctypes.data, res.ctypes.data, pup.ctypes.data, C.byref(lag)))
    del keep
    return hr, res, pup, lag.value


class PendingReconstruction:
    """An in-flight fpmgpu_reconstruct_tiles_async request; wait() returns what
    reconstruct_request returns. Its buffers stay referenced until then."""

    def __init__(self, eng, ticket, keep, out):
        self._eng, self._ticket, self._keep, self._out = eng, ticket, keep, out

    def wait(self):
        lag = C.c_int()
        check(lib().fpmgpu_wait(self._eng.handle, C.c_longlong(self._ticket), C.byref(lag)))
        self._keep = None
        hr, res, pup = self._out
        return hr, res, pup, lag.value


def pinned_empty(shape, dtype) -> np.ndarray:
    """A numpy array in page-locked host memory (fpmgpu_host_alloc), freed with the array."""
    import weakref
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    ptr = C.c_void_p()
    check(lib().fpmgpu_host_alloc(max(nbytes, 1), C.byref(ptr)))
    buf = (C.c_char * max(nbytes, 1)).from_address(ptr.value)
    weakref.finalize(buf, lib().fpmgpu_host_free, C.c_void_p(ptr.value))
    return np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)


def reconstruct_request_async(req: Request, frames: FrameSet, engine: Engine | None = None) -> PendingReconstruction:
    """fpmgpu_reconstruct_tiles_async: the request's LR upload may overlap the
    previous request's reconstruction (two in flight per engine). The outputs
    live in page-locked memory, so their copies back are asynchronous too."""
    eng = engine or default_engine()
    r, keep = req.c()
    T, n, N = r.num_tiles, req.cfg.tile_size, req.cfg.hr_size()
    imgs = np.ascontiguousarray(frames.images, np.uint16)
    hr = pinned_empty((T, N, N), np.complex64)
    res = pinned_empty((T, req.iters), np.float64)
    pup = pinned_empty((T, n, n), np.complex64)
    t = C.c_longlong()
    check(lib().fpmgpu_reconstruct_tiles_async(eng.handle, C.byref(r), imgs.ctypes.data, imgs.shape[2],
                                               hr.ctypes.data, res.ctypes.data, pup.ctypes.data, C.byref(t)))
    return PendingReconstruction(eng, t.value, (r, keep, imgs), (hr, res, pup))


def reconstruct_tile(frames: FrameSet, tile: TileSpec, cfg: OpticalConfig, iters: int, seq, fft_threads: int = 1,
                     mode: str = "gs", alpha: float = 1.0, beta: float = 1.0,
                     engine: Engine | None = None) -> ReconResult:
    """reconstruct_tile (recon.cpp:141-170); `fft_threads` is accepted for API parity."""
    del fft_threads
    t0 = time.perf_counter()
    req = make_request(frames, cfg, seq, [tile], iters, mode=mode, alpha=alpha, beta=beta)
    hr, res, pup, _ = reconstruct_request(req, frames, engine)
    return ReconResult(hr[0], ReconMetrics(res[0].tolist(), time.perf_counter() - t0), pup[0])


def pipelined_reconstruct_tile(frames: FrameSet, tile: TileSpec, cfg: OpticalConfig, iters: int, seq,
                               lag: int | None = None, force_unsafe: bool = False,
                               engine: Engine | None = None) -> PipelineResult:
    """pipelined_reconstruct_tile (parallel.cpp:52-111): disjoint-disk updates of
    adjacent iteration stages run concurrently in one CTA; bit-identical to the
    sequential kernel at any lag >= min_safe_lag."""
    if iters < 1:
        raise ConfigError("iters must be >= 1")
    t0 = time.perf_counter()
    min_lag = min_safe_lag_tile(seq, tile, cfg)
    use = min_lag if lag is None else int(lag)
    if use < min_lag and not force_unsafe:
        raise UnsafeLagError(f"pipeline lag below the safe minimum of {min_lag}", min_lag)
    req = make_request(frames, cfg, seq, [tile], iters, lag=use, force_unsafe_lag=force_unsafe)
    hr, res, _, used = reconstruct_request(req, frames, engine)
    return PipelineResult(hr[0], ReconMetrics(res[0].tolist(), time.perf_counter() - t0), used, use < min_lag)


def run_offline(frames: FrameSet, cfg: OpticalConfig, seq, opt: RunOptions, engine: Engine | None = None,
                stitch: bool = True) -> RunResult:
    """run_offline (parallel.cpp:155-196): every tile of the FOV in one batched
    launch (one CTA per tile), then the Eq. (1) mosaic."""
    if opt.workers < 1:
        raise ConfigError("workers must be >= 1")
    t0 = time.perf_counter()
    specs = select_tiles(frames, cfg, opt)
    pipeline = opt.force_pipeline or opt.workers > len(specs)
    lag = 0
    if pipeline:
        if opt.mode != "gs":
            raise ConfigError("pipelined schedule requires Gerchberg-Saxton mode")
        lag = -1 if opt.lag is None else int(opt.lag)
    req = make_request(frames, cfg, seq, specs, opt.iters, mode=opt.mode, alpha=opt.alpha, beta=opt.beta,
                       lag=lag, force_unsafe_lag=opt.force_unsafe_lag)
    hr, res, pup, _ = reconstruct_request(req, frames, engine)
    stitched = None
    if stitch and opt.max_tiles is None:
        stitched = stitch_mosaic(hr, specs, cfg, engine)
    wall = time.perf_counter() - t0
    timing = TimingRow("", "offline", opt.workers, 1 if opt.lag is None else opt.lag, len(specs), opt.iters,
                       wall, wall / max(len(specs), 1))
    return RunResult(specs, hr, stitched, timing, [ReconMetrics(r.tolist(), 0.0) for r in res], pup)


def select_tiles(frames: FrameSet, cfg: OpticalConfig, opt: RunOptions) -> list:
    """select_tiles (parallel.cpp:142-153) plus the per-tile defocus extension."""
    specs = partition_tiles(frames.width(), frames.height(), cfg, opt.defocus_um)
    if opt.max_tiles is not None:
        if opt.max_tiles > len(specs):
            raise ConfigError("requested tile count exceeds partition")
        specs = specs[: opt.max_tiles]
    if opt.tile_defocus_um is not None:
        if len(opt.tile_defocus_um) != len(specs):
            raise ConfigError("tile_defocus_um must list one value per tile")
        for s, z in zip(specs, opt.tile_defocus_um):
            s.defocus_um = float(z)
    return specs


def run_online(frames: FrameSet, cfg: OpticalConfig, seq, opt: RunOptions, delay_scale: float = 1.0,
               engine: Engine | None = None, stitch: bool = True) -> RunResult:
    """run_online (parallel.cpp:198-317): frames are replayed against their
    timestamps (scaled by delay_scale); each arrival is copied to the device and
    the first-pass update of every newly complete sequence position runs on all
    tiles at once (fpmgpu_online_push), waiting for the on-axis seed like the
    reference (parallel.cpp:266-273); the remaining iters-1 passes, the HR
    fields and the mosaic follow the stream (parallel.cpp:289-305). Same update
    order as run_offline, hence the same tiles."""
    if opt.workers < 1:
        raise ConfigError("workers must be >= 1")
    if delay_scale < 0:
        raise ConfigError("delay scale must be >= 0")
    t0 = time.perf_counter()
    specs = select_tiles(frames, cfg, opt)
    stream = []
    for led in seq:
        f = frames.find(led)
        if f is None:
            raise DataError("missing frame for a sequence LED")
        stream.append(f)
    req = make_request(frames, cfg, seq, specs, opt.iters, mode=opt.mode, alpha=opt.alpha, beta=opt.beta)
    eng = engine or default_engine()
    r, keep = req.c()
    imgs = np.ascontiguousarray(frames.images, np.uint16)
    ts = (np.zeros(len(frames.leds)) if frames.timestamps is None or len(frames.timestamps) == 0
          else np.asarray(frames.timestamps, np.float64))
    T, n, N = len(specs), cfg.tile_size, cfg.hr_size()
    hr = np.zeros((T, N, N), np.complex64)
    res = np.zeros((T, opt.iters), np.float64)
    pup = np.zeros((T, n, n), np.complex64)
    h = C.c_void_p()
    check(lib().fpmgpu_online_begin(eng.handle, C.byref(r), C.byref(h)))
    try:
        applied = C.c_int()
        pushed = set()
        frame_bytes = imgs.shape[1] * imgs.shape[2] * 2
        for f in stream:  # the ordered frame source (parallel.cpp:220-233)
            wait = t0 + float(ts[f]) * delay_scale - time.perf_counter()
            if wait > 0:
                time.sleep(wait)
            if f in pushed:
                continue
            pushed.add(f)
            check(lib().fpmgpu_online_push(h, f, imgs.ctypes.data + f * frame_bytes, imgs.shape[2],
                                           C.byref(applied)))
        if req.init_frame not in pushed:  # seed outside the sequence: read at stream end
            check(lib().fpmgpu_online_push(h, req.init_frame, imgs.ctypes.data + req.init_frame * frame_bytes,
                                           imgs.shape[2], C.byref(applied)))
        check(lib().fpmgpu_online_finish(h, hr.ctypes.data, res.ctypes.data, pup.ctypes.data))
    finally:
        lib().fpmgpu_online_destroy(h)
        del keep
    acquisition = float(ts[stream[-1]]) * delay_scale if stream else 0.0
    stitched = None
    if stitch and opt.max_tiles is None:
        stitched = stitch_mosaic(hr, specs, cfg, engine)
    wall = time.perf_counter() - t0
    timing = TimingRow("", "online", opt.workers, 1, T, opt.iters, wall, wall / max(T, 1))
    return RunResult(specs, hr, stitched, timing, [ReconMetrics(x.tolist(), 0.0) for x in res], pup, acquisition)


def stitch_mosaic(tiles: np.ndarray, specs: list, cfg: OpticalConfig, engine: Engine | None = None) -> np.ndarray:
    """stitch_mosaic (stitch.cpp:48-86) on the device."""
    eng = engine or default_engine()
    t = np.ascontiguousarray(tiles, np.complex64)
    xy = np.ascontiguousarray([[s.x0, s.y0] for s in specs], np.int32)
    rows, cols = C.c_int(), C.c_int()
    c = cfg.c()
    check(lib().fpmgpu_stitch_mosaic(eng.handle, C.byref(c), t.ctypes.data, xy.ctypes.data, len(xy), None,
                                     C.byref(rows), C.byref(cols)))
    out = np.zeros((rows.value, cols.value), np.complex64)
    check(lib().fpmgpu_stitch_mosaic(eng.handle, C.byref(c), t.ctypes.data, xy.ctypes.data, len(xy),
                                     out.ctypes.data, C.byref(rows), C.byref(cols)))
    return out


# ------------------------------------------------------------------ single-step API
def crop_frame(frame: np.ndarray, tile: TileSpec) -> np.ndarray:
    if tile.y0 + tile.size > frame.shape[0] or tile.x0 + tile.size > frame.shape[1]:
        raise DataError("tile extends past frame bounds")
    return frame[tile.y0:tile.y0 + tile.size, tile.x0:tile.x0 + tile.size]


def init_canvas(frames: FrameSet, tile: TileSpec, cfg: OpticalConfig, engine: Engine | None = None) -> SpectrumCanvas:
    eng = engine or default_engine()
    idx = frames.find(cfg.center_led)
    if idx is None:
        print("fpm: warning: on-axis frame missing, initializing from brightest frame", file=sys.stderr)
        if not frames.leds:
            raise DataError("empty frame set")
        idx = int(np.argmax(frames.images.reshape(len(frames.leds), -1).mean(axis=1)))
    img = np.ascontiguousarray(frames.images[idx], np.uint16)
    N = cfg.hr_size()
    out = np.zeros((N, N), np.complex64)
    c = cfg.c()
    check(lib().fpmgpu_init_canvas(eng.handle, C.byref(c), img.ctypes.data, img.shape[0], img.shape[1],
                                   img.shape[1], tile.x0, tile.y0, out.ctypes.data))
    return SpectrumCanvas(out, cfg)


def canvas_to_field(canvas: SpectrumCanvas, fft_threads: int = 1, engine: Engine | None = None) -> np.ndarray:
    del fft_threads
    eng = engine or default_engine()
    src = np.ascontiguousarray(canvas.spectrum, np.complex64)
    out = np.zeros_like(src)
    c = canvas.cfg.c()
    check(lib().fpmgpu_canvas_to_field(eng.handle, C.byref(c), src.ctypes.data, out.ctypes.data))
    return out


def update_step(canvas: SpectrumCanvas, intensity, wv, pupil: Pupil, fft_threads: int = 1, mode: str = "gs",
                alpha: float = 1.0, beta: float = 1.0, pupil_state: np.ndarray | None = None,
                engine: Engine | None = None) -> float:
    """update_step (recon.cpp:93-134) on the device; EPRY updates `pupil_state`
    (complex64 [n, n], in place) when mode='epry'."""
    del fft_threads
    eng = engine or default_engine()
    n = pupil.grid
    I = np.ascontiguousarray(intensity, np.float32)
    if I.shape != (n, n):
        raise DataError("frame side must equal pupil grid")
    if canvas.spectrum.dtype != np.complex64 or not canvas.spectrum.flags.c_contiguous:
        canvas.spectrum = np.ascontiguousarray(canvas.spectrum, np.complex64)
    P = pupil_state if pupil_state is not None else np.ascontiguousarray(pupil.values, np.complex64)
    res = C.c_double()
    c = canvas.cfg.c()
    check(lib().fpmgpu_update_step(eng.handle, C.byref(c), canvas.spectrum.ctypes.data, I.ctypes.data,
                                   C.c_double(wv[0]), C.c_double(wv[1]), P.ctypes.data, MODES[mode],
                                   C.c_double(alpha), C.c_double(beta), C.byref(res)))
    canvas.updated_offsets.append(spectrum_offset_px(wv, canvas.cfg))
    return res.value


# ------------------------------------------------------------------ device-resident plans
class Plan:
    """fpmgpu_plan: geometry uploaded once; execute() on device buffers (e.g. torch CUDA tensors)."""

    def __init__(self, req: Request, engine: Engine | None = None):
        self.engine = engine or default_engine()
        self.req = req
        r, keep = req.c()
        self._h = C.c_void_p()
        check(lib().fpmgpu_plan_create(self.engine.handle, C.byref(r), C.byref(self._h)))
        del keep
        info = _lib.PlanInfoC()
        check(lib().fpmgpu_plan_get_info(self._h, C.byref(info)))
        self.info = {f[0]: getattr(info, f[0]) for f in _lib.PlanInfoC._fields_}

    def execute(self, frames_ptr: int, row_pitch: int, hr_ptr: int | None, residuals_ptr: int | None,
                pupils_ptr: int | None = None, stream: int | None = None) -> None:
        check(lib().fpmgpu_plan_execute(self._h, frames_ptr, int(row_pitch), hr_ptr, residuals_ptr, pupils_ptr,
                                        stream))

    def execute_mosaic(self, frames_ptr: int, row_pitch: int, mosaic_ptr: int, mosaic_pitch: int,
                       residuals_ptr: int | None, pupils_ptr: int | None = None, stream: int | None = None) -> None:
        """execute() with the HR fields written straight into a mosaic (tiles that
        abut without overlap: stitch_mosaic is a plain placement, stitch.cpp:38).
        mosaic_ptr is the plan's top-left tile position, pitch in complex64 elements."""
        check(lib().fpmgpu_plan_execute_mosaic(self._h, frames_ptr, int(row_pitch), mosaic_ptr, int(mosaic_pitch),
                                               residuals_ptr, pupils_ptr, stream))

    def phase_times(self, reset: bool = True):
        """(ms_init, ms_loop, ms_final) summed over executes since the last reset, and the execute count."""
        ms = (C.c_double * 3)()
        n = C.c_int()
        check(lib().fpmgpu_plan_phase_times(self._h, ms, C.byref(n), int(reset)))
        return (ms[0], ms[1], ms[2]), n.value

    def close(self):
        if self._h:
            lib().fpmgpu_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
