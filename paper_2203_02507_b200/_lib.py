"""ctypes binding of libfpm_b200.so (include/fpm_b200.h).

The library is built in-tree by __graft_entry__.build() (or `make -C
paper_2203_02507_b200/csrc`). There is no fallback: importing an engine call
without the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FPM_B200_LIB=check loads the bounds-checked build (make check: device asserts that
# trap on an out-of-range index; tests/test_gpu_checked.py)
LIB_PATH = os.path.join(_HERE, "lib", "libfpm_b200_check.so" if os.environ.get("FPM_B200_LIB") == "check"
                        else "libfpm_b200.so")

OK, ERR_CONFIG, ERR_DATA, ERR_UNSAFE_LAG, ERR_DOMAIN, ERR_CUDA, ERR_INTERNAL, ERR_UNSUPPORTED = range(8)
MODE_GS, MODE_EPRY = 0, 1
ORDER_SPIRAL, ORDER_RASTER = 0, 1


class FpmError(RuntimeError):
    code = ERR_INTERNAL


class ConfigError(FpmError):
    """fpm::ConfigError (optics.hpp:11-13)."""
    code = ERR_CONFIG


class DataError(FpmError):
    """fpm::DataError (optics.hpp:14-16)."""
    code = ERR_DATA


class UnsafeLagError(FpmError):
    """fpm::UnsafeLagError (parallel.hpp:12-17); .minimum carries the safe lag."""
    code = ERR_UNSAFE_LAG

    def __init__(self, msg: str, minimum: int):
        super().__init__(msg)
        self.minimum = minimum


class DomainError(FpmError, ValueError):
    """std::domain_error (optics.cpp:28-30)."""
    code = ERR_DOMAIN


class CudaError(FpmError):
    code = ERR_CUDA


class UnsupportedError(FpmError):
    code = ERR_UNSUPPORTED


_ERR = {ERR_CONFIG: ConfigError, ERR_DATA: DataError, ERR_DOMAIN: DomainError, ERR_CUDA: CudaError,
        ERR_UNSUPPORTED: UnsupportedError}


class OpticalConfigC(C.Structure):
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


class ReconRequestC(C.Structure):
    _fields_ = [
        ("cfg", OpticalConfigC),
        ("iters", C.c_int), ("mode", C.c_int),
        ("alpha", C.c_double), ("beta", C.c_double),
        ("lag", C.c_int), ("force_unsafe_lag", C.c_int),
        ("num_tiles", C.c_int), ("tile_xy", C.POINTER(C.c_int)),
        ("num_leds", C.c_int), ("offsets", C.POINTER(C.c_int)), ("seq_frame", C.POINTER(C.c_int)),
        ("init_frame", C.c_int),
        ("tile_defocus_um", C.POINTER(C.c_double)),
        ("pupils", C.POINTER(C.c_float)),
        ("num_frames", C.c_int), ("height", C.c_int), ("width", C.c_int),
    ]


class PlanInfoC(C.Structure):
    _fields_ = [
        ("tile_side", C.c_int), ("canvas_side", C.c_int), ("num_tiles", C.c_int), ("num_leds", C.c_int),
        ("iters", C.c_int), ("mode", C.c_int), ("lag", C.c_int), ("groups", C.c_int),
        ("launches_per_execute", C.c_int), ("loop_ctas", C.c_int), ("loop_threads", C.c_int),
        ("loop_smem_bytes", C.c_int), ("updates", C.c_double), ("fft_flops_per_update", C.c_double),
        ("hbm_bytes_per_update", C.c_double), ("support_pixels", C.c_int), ("tiles_abut", C.c_int),
    ]


class MosaicBandInfoC(C.Structure):
    _fields_ = [
        ("rows", C.c_int), ("cols", C.c_int), ("strips", C.c_int), ("strip_lo", C.c_int), ("strip_hi", C.c_int),
        ("row_lo", C.c_int), ("row_hi", C.c_int), ("canvas_side", C.c_int), ("needs_exchange", C.c_int),
    ]


IPC_HANDLE_BYTES = 64


EXPORTS = [
    "fpmgpu_version", "fpmgpu_last_error", "fpmgpu_last_min_lag", "fpmgpu_default_config",
    "fpmgpu_validate_config", "fpmgpu_illumination_wavevector", "fpmgpu_build_pupil",
    "fpmgpu_synthesized_na", "fpmgpu_tile_origins", "fpmgpu_partition_tiles", "fpmgpu_sequence_offsets",
    "fpmgpu_spectrum_offset_px", "fpmgpu_min_safe_lag", "fpmgpu_build_schedule", "fpmgpu_create",
    "fpmgpu_destroy", "fpmgpu_reconstruct_tiles", "fpmgpu_plan_create", "fpmgpu_plan_execute",
    "fpmgpu_plan_destroy", "fpmgpu_plan_get_info", "fpmgpu_plan_phase_times", "fpmgpu_update_step", "fpmgpu_init_canvas",
    "fpmgpu_canvas_to_field", "fpmgpu_stitch_mosaic", "fpmgpu_stitch_mosaic_device",
    "fpmgpu_online_begin", "fpmgpu_online_push", "fpmgpu_online_finish", "fpmgpu_online_destroy",
    "fpmgpu_reconstruct_tiles_async", "fpmgpu_wait", "fpmgpu_plan_execute_mosaic", "fpmgpu_mosaic_band_layout",
    "fpmgpu_mosaic_band_sums", "fpmgpu_mosaic_band_assemble", "fpmgpu_ipc_get_handle", "fpmgpu_ipc_open",
    "fpmgpu_ipc_close", "fpmgpu_host_alloc", "fpmgpu_host_free", "fpmgpu_fft2_c128",
]

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load libfpm_b200.so; raises if it has not been built (no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                              "(make -C paper_2203_02507_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        L.fpmgpu_last_error.restype = C.c_char_p
        L.fpmgpu_plan_execute.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        L.fpmgpu_reconstruct_tiles.argtypes = [C.c_void_p, C.POINTER(ReconRequestC), C.c_void_p, C.c_int64,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
        L.fpmgpu_plan_create.argtypes = [C.c_void_p, C.POINTER(ReconRequestC), C.POINTER(C.c_void_p)]
        L.fpmgpu_reconstruct_tiles_async.argtypes = [C.c_void_p, C.POINTER(ReconRequestC), C.c_void_p, C.c_int64,
                                                     C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_longlong)]
        L.fpmgpu_wait.argtypes = [C.c_void_p, C.c_longlong, C.POINTER(C.c_int)]
        L.fpmgpu_online_begin.argtypes = [C.c_void_p, C.POINTER(ReconRequestC), C.POINTER(C.c_void_p)]
        L.fpmgpu_online_push.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int)]
        L.fpmgpu_online_finish.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.fpmgpu_online_destroy.argtypes = [C.c_void_p]
        L.fpmgpu_plan_destroy.argtypes = [C.c_void_p]
        L.fpmgpu_plan_get_info.argtypes = [C.c_void_p, C.POINTER(PlanInfoC)]
        L.fpmgpu_destroy.argtypes = [C.c_void_p]
        L.fpmgpu_plan_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int]
        L.fpmgpu_update_step.argtypes = [C.c_void_p, C.POINTER(OpticalConfigC), C.c_void_p, C.c_void_p,
                                         C.c_double, C.c_double, C.c_void_p, C.c_int, C.c_double,
                                         C.c_double, C.POINTER(C.c_double)]
        L.fpmgpu_init_canvas.argtypes = [C.c_void_p, C.POINTER(OpticalConfigC), C.c_void_p, C.c_int, C.c_int,
                                         C.c_int64, C.c_int, C.c_int, C.c_void_p]
        L.fpmgpu_canvas_to_field.argtypes = [C.c_void_p, C.POINTER(OpticalConfigC), C.c_void_p, C.c_void_p]
        L.fpmgpu_stitch_mosaic.argtypes = [C.c_void_p, C.POINTER(OpticalConfigC), C.c_void_p, C.c_void_p,
                                           C.c_int, C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.fpmgpu_stitch_mosaic_device.argtypes = [C.c_void_p, C.POINTER(OpticalConfigC), C.c_void_p, C.c_void_p,
                                                  C.c_int, C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                                  C.c_void_p]
        L.fpmgpu_plan_execute_mosaic.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                                 C.c_void_p, C.c_void_p, C.c_void_p]
        L.fpmgpu_mosaic_band_layout.argtypes = [C.POINTER(OpticalConfigC), C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                C.POINTER(MosaicBandInfoC)]
        L.fpmgpu_mosaic_band_sums.argtypes = [C.c_void_p, C.POINTER(OpticalConfigC), C.c_void_p, C.c_int, C.c_int,
                                              C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.fpmgpu_mosaic_band_assemble.argtypes = [C.c_void_p, C.POINTER(OpticalConfigC), C.c_void_p, C.c_int,
                                                  C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_int64, C.c_void_p]
        L.fpmgpu_ipc_get_handle.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
        L.fpmgpu_ipc_open.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.fpmgpu_ipc_close.argtypes = [C.c_void_p, C.c_void_p]
        L.fpmgpu_host_alloc.argtypes = [C.c_int64, C.POINTER(C.c_void_p)]
        L.fpmgpu_host_free.argtypes = [C.c_void_p]
        L.fpmgpu_fft2_c128.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    L = lib()
    msg = L.fpmgpu_last_error().decode()
    if rc == ERR_UNSAFE_LAG:
        raise UnsafeLagError(msg, L.fpmgpu_last_min_lag())
    raise _ERR.get(rc, FpmError)(msg)
