"""Tile sharding over GPUs (config 4/5): one process per GPU, no collective in
the reconstruction; the only exchanges build the final mosaic.

Tiles share nothing (run_offline's pool, parallel.cpp:167-181),
so rank r takes a contiguous band of tile rows and only the LR rows that band
covers. The band is expressed as an ordinary Request on the cropped stack, so
each rank runs the single-GPU plan unchanged.

The mosaic (stitch_mosaic, stitch.cpp:48-86, inside run_offline's wall clock at
parallel.cpp:183) is built band by band, every rank writing its own mosaic rows
into rank 0's buffer over NVLink (CUDA IPC peer pointer, no NCCL in the data
path):
  * tiles that abut without overlap (BASELINE configs 3-5, ov = 0): Eq. (1)
    is a plain placement, so canvas_to_field writes each HR field straight into
    the peer mosaic (Plan.execute_mosaic);
  * overlapping tiles: each band forms its strips' ratios and row sums on its
    GPU (fpmgpu_mosaic_band_sums), the ranks combine the [strips][N] sums with
    one all-reduce (zero-filled elsewhere, so the sum is exact), and each band
    assembles its rows (fpmgpu_mosaic_band_assemble) — the same arithmetic as the
    single-GPU stitch_mosaic, hence the same bits.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from ._lib import check, lib
from .engine import Engine, Request


def tile_row_bands(rows: int, world: int) -> list:
    """[(lo, hi)) tile-row ranges, contiguous, balanced to within one row."""
    return [((rows * r) // world, (rows * (r + 1)) // world) for r in range(world)]


@dataclass
class Shard:
    rank: int
    tiles: np.ndarray      # indices into the full request's tile list (a contiguous range)
    y_lo: int              # first LR row of the band in the full stack
    y_hi: int              # one past the last LR row
    request: Request       # the band's request on frames[:, y_lo:y_hi, :]

    @property
    def tile_lo(self) -> int:
        return int(self.tiles[0])

    @property
    def tile_hi(self) -> int:
        return int(self.tiles[-1]) + 1


def shard_request(full: Request, rank: int, world: int) -> Shard:
    """Contiguous tile-row band of `rank`. Tile rows are the distinct y origins
    of the (row-major) partition; the band's stack rows cover every tile in it."""
    ys = np.unique(full.tile_xy[:, 1])
    lo, hi = tile_row_bands(len(ys), world)[rank]
    mine = np.nonzero(np.isin(full.tile_xy[:, 1], ys[lo:hi]))[0]
    if len(mine) == 0:
        raise ValueError(f"rank {rank} of {world} has no tile rows ({len(ys)} rows)")
    if not np.array_equal(mine, np.arange(mine[0], mine[-1] + 1)):
        raise ValueError("tile rows must be contiguous in the tile list (row-major partition)")
    n = full.cfg.tile_size
    y_lo = int(full.tile_xy[mine, 1].min())
    y_hi = int(full.tile_xy[mine, 1].max()) + n
    xy = full.tile_xy[mine].copy()
    xy[:, 1] -= y_lo
    req = replace(full, tile_xy=xy, offsets=full.offsets[mine], height=y_hi - y_lo,
                  tile_defocus_um=None if full.tile_defocus_um is None else full.tile_defocus_um[mine],
                  pupils=None if full.pupils is None else full.pupils[mine])
    return Shard(rank, mine, y_lo, y_hi, req)


def gather_tiles(local, shards: list, rank: int, full_shape, device=None, out=None):
    """Gather every rank's HR tiles to rank 0 (point-to-point over the process
    group: NCCL over NVLink on the B200 box, gloo in the CPU tests). All receives
    are posted together and land straight in their contiguous slice of `out`.
    Returns the full [T, ...] tensor on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist
    if rank != 0:
        dist.send(local.contiguous(), dst=0)
        return None
    if out is None:
        out = torch.empty(full_shape, dtype=local.dtype, device=device if device is not None else local.device)
    out[shards[0].tile_lo:shards[0].tile_hi] = local
    ops = [dist.P2POp(dist.irecv, out[s.tile_lo:s.tile_hi], s.rank) for s in shards[1:]]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return out


# ------------------------------------------------------------------ mosaic bands
@dataclass
class BandLayout:
    rows: int
    cols: int
    strips: int
    strip_lo: int
    strip_hi: int
    row_lo: int
    row_hi: int
    canvas_side: int
    needs_exchange: bool


def band_layout(cfg, xy_all: np.ndarray, tile_lo: int, tile_hi: int) -> BandLayout:
    """Geometry of one band of the FOV's mosaic (host only)."""
    xy = np.ascontiguousarray(xy_all, np.int32)
    info = _lib.MosaicBandInfoC()
    c = cfg.c()
    check(lib().fpmgpu_mosaic_band_layout(C.byref(c), xy.ctypes.data, len(xy), int(tile_lo), int(tile_hi),
                                          C.byref(info)))
    return BandLayout(info.rows, info.cols, info.strips, info.strip_lo, info.strip_hi, info.row_lo, info.row_hi,
                      info.canvas_side, bool(info.needs_exchange))


def stitch_band(engine: Engine, cfg, xy_all: np.ndarray, tile_lo: int, tile_hi: int, tiles_ptr: int,
                mosaic_ptr: int, mosaic_pitch: int, combine=None, stream: int | None = None) -> BandLayout:
    """Write this band's rows of the FOV's Eq. (1) mosaic into mosaic_ptr (row 0
    of the whole mosaic, possibly a peer GPU's buffer). tiles_ptr: the band's HR
    tiles on this GPU [tile_hi - tile_lo][N][N] complex64. combine(sums) -> sums
    must return the element-wise sum of every band's [strips][N][2] float64
    array (an all-reduce; identity for one band). Returns after the rows are written."""
    lay = band_layout(cfg, xy_all, tile_lo, tile_hi)
    xy = np.ascontiguousarray(xy_all, np.int32)
    c = cfg.c()
    sums = np.zeros((lay.strips, lay.canvas_side, 2), np.float64)
    ratios = np.zeros((tile_hi - tile_lo, 2), np.float64)
    check(lib().fpmgpu_mosaic_band_sums(engine.handle, C.byref(c), xy.ctypes.data, len(xy), int(tile_lo),
                                        int(tile_hi), tiles_ptr, sums.ctypes.data, ratios.ctypes.data, stream))
    if lay.needs_exchange and combine is not None:
        sums = np.ascontiguousarray(combine(sums), np.float64)
    check(lib().fpmgpu_mosaic_band_assemble(engine.handle, C.byref(c), xy.ctypes.data, len(xy), int(tile_lo),
                                            int(tile_hi), tiles_ptr, sums.ctypes.data, ratios.ctypes.data,
                                            mosaic_ptr, int(mosaic_pitch), stream))
    return lay


def allreduce_sum(device=None):
    """combine() for stitch_band over the default process group: one all-reduce
    of the zero-filled strip sums (on `device` for NCCL, on the host for gloo)."""
    import torch
    import torch.distributed as dist

    def combine(a: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(a))
        if device is not None:
            t = t.to(device)
        dist.all_reduce(t)
        return t.cpu().numpy()
    return combine


class PeerMosaic:
    """Rank 0's mosaic buffer opened in every rank's process (CUDA IPC; over
    NVLink / NVSwitch between GPUs). `ptr` is the mosaic's row 0 on this rank:
    rank 0's own pointer there, the opened peer mapping elsewhere."""

    def __init__(self, engine: Engine, rank: int, local_ptr: int | None, broadcast):
        """local_ptr: rank 0's device buffer (ignored elsewhere); broadcast(obj)
        -> obj must deliver rank 0's object to every rank (e.g. broadcast_object_list)."""
        self.engine = engine
        self._opened = None
        if rank == 0:
            h = (C.c_ubyte * _lib.IPC_HANDLE_BYTES)()
            off = C.c_int64()
            check(lib().fpmgpu_ipc_get_handle(C.c_void_p(local_ptr), h, C.byref(off)))
            broadcast((bytes(h), off.value))
            self.ptr = int(local_ptr)
        else:
            raw, off = broadcast(None)
            h = (C.c_ubyte * _lib.IPC_HANDLE_BYTES).from_buffer_copy(raw)
            p = C.c_void_p()
            check(lib().fpmgpu_ipc_open(engine.handle, h, C.byref(p)))
            self._opened = p.value
            self.ptr = int(p.value) + int(off)

    def close(self):
        if self._opened:
            check(lib().fpmgpu_ipc_close(self.engine.handle, C.c_void_p(self._opened)))
            self._opened = None


def broadcast_from_rank0(device=None):
    """broadcast() for PeerMosaic over the default process group."""
    import torch.distributed as dist

    def bcast(obj):
        box = [obj]
        dist.broadcast_object_list(box, src=0, device=device)
        return box[0]
    return bcast
