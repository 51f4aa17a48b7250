"""Tile sharding over GPUs (config 4/5): one process per GPU, no collective in
the reconstruction; the only exchange is the final HR gather to rank 0.

Tiles share nothing (run_offline's pool, parallel.cpp:167-181),
so rank r takes a contiguous band of tile rows and only the LR rows that band
covers. The band is expressed as an ordinary Request on the cropped stack, so
each rank runs the single-GPU plan unchanged.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .engine import Request


def tile_row_bands(rows: int, world: int) -> list:
    """[(lo, hi)) tile-row ranges, contiguous, balanced to within one row."""
    return [((rows * r) // world, (rows * (r + 1)) // world) for r in range(world)]


@dataclass
class Shard:
    rank: int
    tiles: np.ndarray      # indices into the full request's tile list
    y_lo: int              # first LR row of the band in the full stack
    y_hi: int              # one past the last LR row
    request: Request       # the band's request on frames[:, y_lo:y_hi, :]


def shard_request(full: Request, rank: int, world: int) -> Shard:
    """Contiguous tile-row band of `rank`. Tile rows are the distinct y origins
    of the (row-major) partition; the band's stack rows cover every tile in it."""
    ys = np.unique(full.tile_xy[:, 1])
    lo, hi = tile_row_bands(len(ys), world)[rank]
    mine = np.nonzero(np.isin(full.tile_xy[:, 1], ys[lo:hi]))[0]
    if len(mine) == 0:
        raise ValueError(f"rank {rank} of {world} has no tile rows ({len(ys)} rows)")
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
    group: NCCL over NVLink on the B200 box, gloo in the CPU tests). Returns the
    full [T, ...] tensor on rank 0 (into `out` when given), None elsewhere."""
    import torch
    import torch.distributed as dist
    if rank != 0:
        dist.send(local.contiguous(), dst=0)
        return None
    if out is None:
        out = torch.empty(full_shape, dtype=local.dtype, device=device if device is not None else local.device)
    idx0 = torch.as_tensor(shards[0].tiles, device=out.device)
    out[idx0] = local
    for s in shards[1:]:
        buf = torch.empty((len(s.tiles),) + tuple(full_shape[1:]), dtype=local.dtype, device=out.device)
        dist.recv(buf, src=s.rank)
        out[torch.as_tensor(s.tiles, device=out.device)] = buf
    return out
