"""Multi-GPU host logic on CPU (gloo, world_size 2 and 3): tile-row sharding of
the config-3/4 geometry and the HR gather to rank 0. The device kernels are
covered by the GPU tests; this checks that every tile is reconstructed exactly
once, from the right rows of the band, and lands in its place on rank 0."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2203_02507_b200 as fpm
from paper_2203_02507_b200.distributed import (allreduce_sum, band_layout, gather_tiles, shard_request,
                                               tile_row_bands)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _full_request(fov=2048):
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=0, led_scan_rows=15, led_scan_cols=15)
    seq = fpm.led_sequence("spiral", cfg)
    xy, _, _, of = fpm.partition_arrays(fov, fov, cfg, seq)
    defocus = np.random.default_rng(7).uniform(-10, 10, len(xy))
    return fpm.Request(cfg, 10, xy, of, np.arange(len(seq), dtype=np.int32), 0, len(seq), fov, fov, mode="epry",
                       tile_defocus_um=defocus)


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = _full_request()
    T = len(full.tile_xy)
    shards = [shard_request(full, r, world) for r in range(world)]
    me = shards[rank]
    # the band's request is the full request restricted to my tiles, y-shifted
    assert np.array_equal(me.request.offsets, full.offsets[me.tiles])
    assert np.array_equal(me.request.tile_xy[:, 0], full.tile_xy[me.tiles, 0])
    assert np.array_equal(me.request.tile_xy[:, 1] + me.y_lo, full.tile_xy[me.tiles, 1])
    assert np.array_equal(me.request.tile_defocus_um, full.tile_defocus_um[me.tiles])
    assert me.request.height == me.y_hi - me.y_lo
    # every crop of the band equals the full-stack crop at the original position
    stack = np.arange(2 * full.height * full.width, dtype=np.int64).reshape(2, full.height, full.width) % 65521
    band = stack[:, me.y_lo:me.y_hi, :]
    for i in (0, len(me.tiles) - 1):
        x0, y0 = me.request.tile_xy[i]
        X0, Y0 = full.tile_xy[me.tiles[i]]
        assert np.array_equal(band[:, y0:y0 + 64, x0:x0 + 64], stack[:, Y0:Y0 + 64, X0:X0 + 64])
    # stand-in HR tiles: value = global tile index; gather to rank 0
    local = torch.as_tensor(me.tiles, dtype=torch.float32)[:, None, None].expand(len(me.tiles), 4, 4).contiguous()
    out = gather_tiles(local, shards, rank, (T, 4, 4))
    if rank == 0:
        ok = bool(torch.equal(out[:, 0, 0], torch.arange(T, dtype=torch.float32)))
        result_q.put(("ok", ok, [len(s.tiles) for s in shards]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tile_sharding_and_gather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    tag, ok, sizes = q.get(timeout=10)
    assert ok
    assert sum(sizes) == 1024 and max(sizes) - min(sizes) <= 32  # balanced to one tile row


def test_tile_row_bands_cover_once():
    for rows in (1, 7, 32, 18):
        for world in (1, 2, 3, 4, 8):
            if world > rows:
                continue
            b = tile_row_bands(rows, world)
            assert b[0][0] == 0 and b[-1][1] == rows
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1


def _layout_worker(rank, world, port, fov, n, ov, result_q):
    """Each rank's mosaic band: rows and strips partition the mosaic; the strip-sum
    exchange (zero-filled all-reduce) reproduces every band's sums exactly."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = fpm.OpticalConfig(tile_size=n, tile_overlap=ov, led_scan_rows=3, led_scan_cols=3)
    seq = fpm.led_sequence("spiral", cfg)
    xy, _, _, of = fpm.partition_arrays(fov, fov, cfg, seq)
    full = fpm.Request(cfg, 1, xy, of, np.arange(len(seq), dtype=np.int32), 0, len(seq), fov, fov)
    me = shard_request(full, rank, world)
    lay = band_layout(cfg, xy, me.tile_lo, me.tile_hi)
    whole = band_layout(cfg, xy, 0, len(xy))
    # stand-in strip sums: band-owned strips hold (strip, row) codes, the rest zeros
    sums = np.zeros((lay.strips, lay.canvas_side, 2))
    for s_ in range(lay.strip_lo, lay.strip_hi):
        sums[s_, :, 0] = s_ + np.arange(lay.canvas_side) / 7.0
        sums[s_, :, 1] = -s_
    got = allreduce_sum()(sums)
    want = np.zeros_like(sums)
    for s_ in range(lay.strips):
        want[s_, :, 0] = s_ + np.arange(lay.canvas_side) / 7.0
        want[s_, :, 1] = -s_
    ok = bool(np.array_equal(got, want))
    rec = [None] * world
    dist.all_gather_object(rec, (lay.row_lo, lay.row_hi, lay.strip_lo, lay.strip_hi, lay.rows, lay.cols,
                                 lay.needs_exchange))
    if rank == 0:
        result_q.put((ok, rec, (whole.rows, whole.cols, whole.strips, whole.needs_exchange)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,fov,n,ov", [(2, 2048, 64, 0), (3, 2048, 64, 0), (2, 240, 64, 8), (3, 500, 64, 12)])
def test_mosaic_bands_partition_gloo(world, fov, n, ov):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_layout_worker, args=(r, world, port, fov, n, ov, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    ok, rec, (rows, cols, strips, exch) = q.get(timeout=10)
    assert ok
    assert exch == (ov > 0)
    # every mosaic row and every strip belongs to exactly one band, in rank order
    assert rec[0][0] == 0 and rec[-1][1] == rows and rec[0][2] == 0 and rec[-1][3] == strips
    for a, b in zip(rec, rec[1:]):
        assert a[1] == b[0] and a[3] == b[2]
    assert all(r[4] == rows and r[5] == cols and r[6] == exch for r in rec)
    assert rows == cols == 4 * fov


def test_mosaic_band_must_be_whole_rows():
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=0, led_scan_rows=3, led_scan_cols=3)
    xy, _, _, _ = fpm.partition_arrays(256, 256, cfg, fpm.led_sequence("spiral", cfg))
    band_layout(cfg, xy, 4, 8)
    with pytest.raises(fpm.DataError, match="whole tile rows"):
        band_layout(cfg, xy, 2, 6)
