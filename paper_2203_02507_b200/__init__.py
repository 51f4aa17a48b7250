"""B200-native Fourier-ptychography reconstruction engine (arxiv 2203.02507 hot path).

The reference's per-tile reconstruction API (reconstruct_tile,
pipelined_reconstruct_tile, run_offline, update_step) over libfpm_b200.so:
hand-written sm_100a kernels behind a C-ABI (include/fpm_b200.h).
"""
from .engine import (ConfigError, DataError, DomainError, Engine, FrameSet, OpticalConfig, Plan,  # noqa: F401
                     Pupil, ReconResult, Request, RunOptions, RunResult, SpectrumCanvas, TileSpec,
                     UnsafeLagError, build_pupil, build_schedule, canvas_to_field, crop_frame, default_engine,
                     illumination_wavevector, init_canvas, led_sequence, make_request, min_safe_lag,
                     min_safe_lag_tile, partition_arrays, partition_tiles, pipelined_reconstruct_tile,
                     reconstruct_request, reconstruct_request_async, reconstruct_tile, run_offline, run_online, scan_leds, select_tiles, sequence_offsets,
                     spectrum_offset_px, stitch_mosaic, synthesized_na, tile_origins, update_step)

from ._lib import CudaError, UnsupportedError  # noqa: F401,E402
from .engine import pinned_empty  # noqa: F401,E402
from .forward import simulate_dataset  # noqa: F401,E402
from .formats import (AppConfig, Dataset, IoError, NoiseSpec, RunConfig, config_from_json,  # noqa: F401,E402
                      config_to_json, export_view, import_view, read_cfi, read_config, read_dataset, read_pgm16,
                      write_cfi, write_config, write_dataset, write_pgm16)

__all__ = [n for n in dir() if not n.startswith("_")]
