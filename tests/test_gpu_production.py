"""GPU parity of the exact kernel paths the BASELINE configurations run in
production (bench.py), and of the mosaic paths (single GPU and multi-rank).

* config 5's production loop: n = 256 tiles, 21x21 LEDs, 10 EPRY iterations,
  per-tile defocus, 4-CTA clusters with the persistent cluster work queue;
* config 3's bench plan: one Plan.execute over all 1,024 tiles on a device
  stack (persistent work queue with parts), bit-identical to run_offline's
  banded host path and within the north star's 1e-3 of the oracle;
* the fused mosaic write (Plan.execute_mosaic) against execute + stitch;
* the multi-rank mosaic: two processes (gloo for the host exchange, CUDA IPC for
  the peer mosaic) each writing its band of rank 0's mosaic, bit-identical to
  the single-GPU stitch_mosaic — overlapping tiles (strip-sum exchange) and
  abutting tiles (execute_mosaic into the peer buffer).
"""
import os
import socket

import numpy as np
import pytest

import paper_2203_02507_b200 as fpm
from tests.helpers import amp_phase_rel, dataset, gpu_cfg, orc_cfg

pytestmark = pytest.mark.gpu

FINAL_TOL = 1e-3


def test_config5_production_path_full_count(orc, monkeypatch):
    """BASELINE config 5's kernel path at full iteration count: 4 tiles of
    256x256 LR (N = 1024), 21x21 LEDs, 10 EPRY iterations, per-tile defocus, on
    4-CTA clusters with the cluster work queue forced (FPM_B200_QUEUE=1: a grid
    of clusters wider than the tile count, as when 256 tiles share 74 resident
    clusters). Two tiles against the oracle's reconstruct_tile
    (recon.cpp:161-167) at the north star's 1e-3."""
    import torch
    from paper_2203_02507_b200.forward import simulate_dataset
    cfg = fpm.OpticalConfig(tile_size=256, tile_overlap=0, upsample=4, led_scan_rows=21, led_scan_cols=21)
    oc = orc_cfg(cfg)
    obj = orc.synth_object("composite", 2048, 17)
    seq = orc.led_sequence("spiral", oc)
    fs = simulate_dataset(obj, seq, cfg, defocus_um=5.0, device="cuda")
    assert fs.images.shape == (441, 512, 512)
    torch.cuda.empty_cache()
    dz = [7.5, -4.0, 2.0, -9.0]
    monkeypatch.setenv("FPM_B200_CLUSTER", "4")
    monkeypatch.setenv("FPM_B200_QUEUE", "1")
    monkeypatch.setenv("FPM_B200_BANDS", "1")
    got = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=10, mode="epry", tile_defocus_um=dz),
                          engine=fpm.Engine(0), stitch=False)
    assert got.tiles.shape == (4, 1024, 1024)
    ofs = orc.FrameStack(fs.images, list(fs.leds))
    for t in (0, 3):
        ref = orc.reconstruct_tile(ofs, oc, 10, seq, tile_index=t, mode="epry", tile_defocus=dz[t])
        amp, ph = amp_phase_rel(got.tiles[t], ref.hr)
        print(f"config 5 production path, tile {t}: amplitude rel-L2 {amp:.2e}, phase {ph:.2e}")
        assert amp < FINAL_TOL and ph < FINAL_TOL, (t, amp, ph)
        # per-pass residuals: the first pass at 1e-3; later passes average per-LED ratios whose
        # dark-field denominators (21x21 scan at n = 256) amplify FP32-vs-FP64 rounding, 1e-2
        res = np.asarray(got.tile_metrics[t].pass_mean_residual)
        assert np.allclose(res[0], ref.residuals[0], rtol=1e-3)
        assert np.allclose(res, ref.residuals, rtol=1e-2)


def test_config3_bench_plan_exact(orc):
    """bench.py's exact plan: the config-3 request (1,024 tiles, 15x15 LEDs, 10
    EPRY iterations, per-tile defocus seed 7) built the way bench.py builds it,
    one Plan.execute on a device stack (1,024 tiles > 592 resident CTAs: the
    persistent work queue with parts serves it). Its tiles and residuals equal
    run_offline's (the banded host path, queue off) bit for bit; three tiles
    match the oracle at 1e-3; and execute_mosaic (the bench step) writes the
    same fields into the FOV mosaic."""
    import torch
    from paper_2203_02507_b200.forward import simulate_dataset
    cfg = fpm.OpticalConfig(tile_size=64, tile_overlap=0, upsample=4, led_scan_rows=15, led_scan_cols=15)
    oc = orc_cfg(cfg)
    obj = orc.synth_object("composite", 8192, 23)
    seq = fpm.led_sequence("spiral", cfg)
    fs = simulate_dataset(obj, seq, cfg, defocus_um=-4.0, device="cuda")
    L, F = len(seq), 2048
    assert fs.images.shape == (L, F, F) and [tuple(x) for x in fs.leds] == [tuple(x) for x in seq]
    xy, _, _, of = fpm.partition_arrays(F, F, cfg, seq)
    defocus = np.random.default_rng(7).uniform(-10.0, 10.0, len(xy))
    req = fpm.Request(cfg, 10, xy, of, np.arange(L, dtype=np.int32), 0, L, F, F, mode="epry",
                      tile_defocus_um=defocus)
    dev = torch.device("cuda", 0)
    frames = torch.from_numpy(fs.images).to(dev)
    eng = fpm.Engine(0)
    plan = fpm.Plan(req, eng)
    assert plan.info["num_tiles"] == 1024 and plan.info["tiles_abut"] == 1
    hr = torch.empty((1024, 256, 256, 2), dtype=torch.float32, device=dev)
    res = torch.empty((1024, 10), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    plan.execute(frames.data_ptr(), F, hr.data_ptr(), res.data_ptr(), None, s.cuda_stream)
    mosaic = torch.empty((8192, 8192, 2), dtype=torch.float32, device=dev)
    res2 = torch.empty_like(res)
    plan.execute_mosaic(frames.data_ptr(), F, mosaic.data_ptr(), 8192, res2.data_ptr(), None, s.cuda_stream)
    torch.cuda.synchronize()
    tiles = hr.cpu().numpy().view(np.complex64)[..., 0]
    resid = res.cpu().numpy()
    assert np.array_equal(resid, res2.cpu().numpy())
    mos = mosaic.cpu().numpy().view(np.complex64)[..., 0]
    for t in range(1024):
        x0, y0 = xy[t]
        assert np.array_equal(mos[4 * y0:4 * y0 + 256, 4 * x0:4 * x0 + 256], tiles[t]), t
    del hr, mosaic, frames
    torch.cuda.empty_cache()
    ref = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=10, mode="epry", tile_defocus_um=list(defocus)),
                          engine=eng, stitch=False)
    assert np.array_equal(ref.tiles, tiles)
    assert np.array_equal(np.array([m.pass_mean_residual for m in ref.tile_metrics]), resid)
    ofs = orc.FrameStack(fs.images, list(fs.leds))
    for t in (5, 480, 1023):
        o = orc.reconstruct_tile(ofs, oc, 10, seq, tile_index=t, mode="epry", tile_defocus=float(defocus[t]))
        amp, ph = amp_phase_rel(tiles[t], o.hr)
        assert amp < FINAL_TOL and ph < FINAL_TOL, (t, amp, ph)
        assert np.allclose(resid[t], o.residuals, rtol=1e-3)


def test_execute_mosaic_equals_execute_then_stitch(eng):
    """Abutting tiles (overlap 0): canvas_to_field written straight into the
    mosaic gives stitch_mosaic's bits (a plain placement, stitch.cpp:38); tiles
    that overlap are refused with the reference's data-error family."""
    import torch
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=0)
    fs, _, seq, _ = dataset(cfg, fov=256, seed=71)
    specs = fpm.partition_tiles(256, 256, cfg)
    for t, d in zip(specs, np.linspace(-6, 6, len(specs))):
        t.defocus_um = float(d)
    req = fpm.make_request(fs, cfg, seq, specs, 2, mode="epry")
    dev = torch.device("cuda", 0)
    frames = torch.from_numpy(np.ascontiguousarray(fs.images)).to(dev)
    plan = fpm.Plan(req, eng)
    hr = torch.empty((16, 256, 256, 2), dtype=torch.float32, device=dev)
    res = torch.empty((16, 2), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    plan.execute(frames.data_ptr(), 256, hr.data_ptr(), res.data_ptr(), None, s)
    torch.cuda.synchronize()
    stitched = fpm.stitch_mosaic(hr.cpu().numpy().view(np.complex64)[..., 0], specs, cfg, eng)
    mosaic = torch.full((1024, 1030, 2), 7.0, dtype=torch.float32, device=dev)  # pitch wider than the mosaic
    plan.execute_mosaic(frames.data_ptr(), 256, mosaic.data_ptr(), 1030, res.data_ptr(), None, s)
    torch.cuda.synchronize()
    m = mosaic.cpu().numpy().view(np.complex64)[..., 0]
    assert np.array_equal(m[:, :1024], stitched)
    assert np.all(m[:, 1024:] == 7.0 + 7.0j)
    cfg8 = gpu_cfg(led_scan_rows=3, led_scan_cols=3, tile_overlap=8)
    fs8, _, seq8, _ = dataset(cfg8, fov=120, seed=72)
    p8 = fpm.Plan(fpm.make_request(fs8, cfg8, seq8, fpm.partition_tiles(120, 120, cfg8), 1), eng)
    assert p8.info["tiles_abut"] == 0
    with pytest.raises(fpm.UnsupportedError, match="overlap"):
        p8.execute_mosaic(frames.data_ptr(), 120, mosaic.data_ptr(), 1030, res.data_ptr(), None, s)


# ------------------------------------------------------------------ multi-rank mosaic
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tiles_for(fov, n, ov, seed):
    cfg = fpm.OpticalConfig(tile_size=n, tile_overlap=ov, upsample=4, led_scan_rows=3, led_scan_cols=3)
    xy, _, _, _ = fpm.partition_arrays(fov, fov, cfg, fpm.led_sequence("spiral", cfg))
    rng = np.random.default_rng(seed)
    N = 4 * n
    t = (1.0 + 0.3 * rng.standard_normal((len(xy), N, N)) + 0.3j * rng.standard_normal((len(xy), N, N)))
    t *= np.exp(1j * rng.uniform(-np.pi, np.pi, (len(xy), 1, 1)))  # per-tile phase: the ratios matter
    return cfg, xy, t.astype(np.complex64)


def _mosaic_worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    from paper_2203_02507_b200.distributed import (PeerMosaic, allreduce_sum, band_layout, broadcast_from_rank0,
                                                   shard_request, stitch_band)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    eng = fpm.Engine(0)
    try:
        if case == "overlap":
            cfg, xy, tiles = _tiles_for(240, 64, 8, seed=5)
            seq = fpm.led_sequence("spiral", cfg)
            full = fpm.Request(cfg, 1, xy, np.zeros((len(xy), len(seq), 2), np.int32),
                               np.arange(len(seq), dtype=np.int32), 0, len(seq), 240, 240)
            me = shard_request(full, rank, world)
            lay = band_layout(cfg, xy, me.tile_lo, me.tile_hi)
            mosaic = torch.zeros((lay.rows, lay.cols, 2), dtype=torch.float32, device=dev) if rank == 0 else None
            peer = PeerMosaic(eng, rank, mosaic.data_ptr() if rank == 0 else None, broadcast_from_rank0())
            band = torch.from_numpy(tiles[me.tile_lo:me.tile_hi].view(np.float32)).to(dev)
            stitch_band(eng, cfg, xy, me.tile_lo, me.tile_hi, band.data_ptr(), peer.ptr, lay.cols, allreduce_sum())
            torch.cuda.synchronize()
            dist.barrier()
            if rank == 0:
                ref = fpm.stitch_mosaic(tiles, [fpm.TileSpec(int(a), int(b), 64) for a, b in xy], cfg, eng)
                got = mosaic.cpu().numpy().view(np.complex64)[..., 0]
                q.put(("overlap", bool(np.array_equal(got, ref)), lay.needs_exchange))
        else:  # abutting tiles: each band's canvas_to_field writes rank 0's mosaic over the peer pointer
            cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=0)
            fs, _, seq, _ = dataset(cfg, fov=256, seed=73)
            specs = fpm.partition_tiles(256, 256, cfg)
            for t, d in zip(specs, np.linspace(-5, 5, len(specs))):
                t.defocus_um = float(d)
            full = fpm.make_request(fs, cfg, seq, specs, 2, mode="epry")
            me = shard_request(full, rank, world)
            lay = band_layout(cfg, full.tile_xy, me.tile_lo, me.tile_hi)
            mosaic = torch.zeros((lay.rows, lay.cols, 2), dtype=torch.float32, device=dev) if rank == 0 else None
            peer = PeerMosaic(eng, rank, mosaic.data_ptr() if rank == 0 else None, broadcast_from_rank0())
            frames = torch.from_numpy(np.ascontiguousarray(fs.images[:, me.y_lo:me.y_hi, :])).to(dev)
            plan = fpm.Plan(me.request, eng)
            res = torch.empty((len(me.tiles), 2), dtype=torch.float64, device=dev)
            s = torch.cuda.current_stream(dev).cuda_stream
            plan.execute_mosaic(frames.data_ptr(), 256, peer.ptr + lay.row_lo * lay.cols * 8, lay.cols,
                                res.data_ptr(), None, s)
            torch.cuda.synchronize()
            dist.barrier()
            if rank == 0:
                whole = fpm.Plan(full, eng)
                ff = torch.from_numpy(np.ascontiguousarray(fs.images)).to(dev)
                ref = torch.zeros_like(mosaic)
                r2 = torch.empty((len(specs), 2), dtype=torch.float64, device=dev)
                whole.execute_mosaic(ff.data_ptr(), 256, ref.data_ptr(), lay.cols, r2.data_ptr(), None, s)
                torch.cuda.synchronize()
                q.put(("abut", bool(torch.equal(mosaic, ref)), lay.needs_exchange))
        dist.barrier()
        peer.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("overlap", 2), ("overlap", 3), ("abut", 2)])
def test_multi_rank_mosaic_over_ipc(case, world):
    """Every rank writes its band of rank 0's mosaic through a CUDA IPC peer
    pointer (the multi-GPU data path; here all ranks share cuda:0, and nothing
    waits on another rank's kernels — the host barrier orders the check). The
    mosaic equals the single-GPU stitch_mosaic / execute_mosaic bit for bit."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mosaic_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    tag, ok, exch = q.get(timeout=10)
    assert tag == case and ok
    assert exch == (case == "overlap")
