"""Benchmark: LED-updates/s of the FPM reconstruction (default: BASELINE config 3/4).

Default workload (config 3, N=1): 2048x2048 sensor, 32x32 tiles of 64x64 LR
px (overlap 0), 15x15 LEDs (spiral order), 10 iterations EPRY, per-tile
illumination k-vectors and per-tile defocus pupils (uniform +-10 um, seed 7);
synthetic u16 LR stack (uniform [0, 52428], seed 1: the cost is
data-independent). One step = one full-FOV reconstruction as run_offline
defines it (parallel.cpp:155-196): pupils + init_canvas + LED loop +
canvas_to_field of every tile + the FOV mosaic (stitch_mosaic). Under torchrun
(N > 1) the default is strong scaling = BASELINE config 4: the FOV is cut into
contiguous tile-row bands, each rank holds only its band of the stack, and
each rank writes its band of rank 0's mosaic over NVLink (CUDA IPC peer
pointer) — the only inter-GPU traffic. `--scaling weak` gives every rank its
own independent FOV instead.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config 3|1|2|5] [--scaling strong|weak] [--no-e2e] [--no-cpu]

`--config` 1/2/5 measure the other BASELINE shapes (single 64 px tile GS;
single 128 px tile EPRY; 4096x4096 sensor of 256 px tiles, 21x21 LEDs).
`--impl reference` times the CPU oracle's restatement of the reference's
multithreaded run_offline (the reference itself cannot be built here: no
Eigen) on a bounded sample of the same workload (one tile row, every
iteration), with every host thread; it loads only oracle/, never the product
library.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "LED-updates/s"


@dataclass(frozen=True)
class Workload:
    key: int
    fov: int
    n: int
    scan: int
    iters: int
    mode: str
    per_tile_defocus: bool
    label: str

    @property
    def tiles(self) -> int:
        return (self.fov // self.n) ** 2

    @property
    def leds(self) -> int:
        return self.scan * self.scan

    @property
    def updates(self) -> int:
        return self.tiles * self.leds * self.iters

    @property
    def stack_bytes(self) -> int:
        return self.leds * self.fov * self.fov * 2

    @property
    def metric(self) -> str:
        return (f"LED-updates/sec ({self.label}: {self.fov}x{self.fov} sensor, {self.tiles} tiles of "
                f"{self.n}x{self.n} LR, {self.scan}x{self.scan} LEDs, {self.iters} iters {self.mode.upper()})")


WORKLOADS = {
    3: Workload(3, 2048, 64, 15, 10, "epry", True, "BASELINE config 3/4 full FOV"),
    1: Workload(1, 64, 64, 15, 10, "gs", False, "BASELINE config 1 single tile"),
    2: Workload(2, 128, 128, 15, 20, "epry", False, "BASELINE config 2 single tile"),
    5: Workload(5, 4096, 256, 21, 10, "epry", True, "BASELINE config 5 large FOV"),
}


def workload_cfg(W: Workload):
    import paper_2203_02507_b200 as fpm
    return fpm.OpticalConfig(tile_size=W.n, tile_overlap=0, upsample=4, led_scan_rows=W.scan, led_scan_cols=W.scan)


def oracle_cfg(W: Workload):
    """The same optics for the CPU legs, built from the oracle alone (the reference
    arm must not load the product library)."""
    from oracle import oracle as orc
    return orc.Optics(tile_size=W.n, tile_overlap=0, upsample=4, led_scan_rows=W.scan, led_scan_cols=W.scan)


def geometry(W: Workload, cfg):
    import paper_2203_02507_b200 as fpm
    seq = fpm.led_sequence("spiral", cfg)
    xy, _, _, of = fpm.partition_arrays(W.fov, W.fov, cfg, seq)
    defocus = np.random.default_rng(7).uniform(-10.0, 10.0, len(xy)) if W.per_tile_defocus else None
    return seq, xy, of, defocus


def l2_flush_needed(W: Workload, world: int) -> bool:
    return W.stack_bytes // max(world, 1) < 256 * 1024 * 1024


def config_block(W: Workload, world: int, scaling: str):
    """The workload block, identical in both arms for the same (N, scaling)."""
    units = W.updates * (world if scaling == "weak" else 1)
    share = world if scaling == "strong" else 1  # ranks sharing one FOV's stack
    return {"workload": f"{W.label}: {W.fov}x{W.fov} sensor, {W.tiles} tiles n={W.n} (N={4 * W.n}), "
                        f"{W.scan}x{W.scan} LEDs spiral, {W.iters} iters {W.mode.upper()}"
                        + (", per-tile k-vectors + defocus pupils" if W.per_tile_defocus else ""),
            "baseline_config": (4 if scaling == "strong" and world > 1 and W.key == 3 else W.key),
            "fov": W.fov, "tile_side": W.n, "canvas_side": 4 * W.n, "leds": W.leds,
            "iters": W.iters, "mode": W.mode, "tiles": W.tiles, "updates_per_step": W.updates,
            "updates_per_step_all_ranks": units, "ranks": world, "sharding": (
                "tile-row bands, one FOV over all ranks" if scaling == "strong" else "one independent FOV per rank"),
            "l2_policy": ("L2 flushed (256 MiB write) between timed steps; per-step CUDA events"
                          if l2_flush_needed(W, share) else
                          f"inputs larger than L2 (LR stack {W.stack_bytes / 2**30:.2f} GiB)")}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            p = [x.strip() for x in l.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU leg (oracle)
def cpu_sample(W: Workload, workers: int):
    """Oracle run_offline on the first tile row of the workload (fov x n crop), one
    iteration, same mode and per-tile defocus; returns (updates/s, wall, tiles).
    Touches only oracle/ (the checker), never the product library."""
    from oracle import oracle as orc
    oc = oracle_cfg(W)
    seq = orc.led_sequence("spiral", oc)
    # a few seconds of work on every host thread, and at most ~15 s in all: the tile rows
    # are capped by a budget of 600 k n = 64-equivalent updates (work ~ n^2 per update)
    per_row = (W.fov // W.n) * W.leds * W.iters * (W.n / 64) ** 2
    rows = max(1, min(W.fov // W.n, workers // 4, int(600_000 // per_row)))
    H = W.n * rows
    rng = np.random.default_rng(1)
    imgs = rng.integers(0, 52429, (len(seq), H, W.fov), dtype=np.uint16)
    fs = orc.FrameStack(imgs, [tuple(l) for l in seq])
    T = (W.fov // W.n) * rows
    if W.mode != "gs":  # the pipelined path (workers > tiles, parallel.cpp:166) is GS-only
        workers = min(workers, T)
    defocus = np.random.default_rng(7).uniform(-10.0, 10.0, 1024 * 1024)[:T] if W.per_tile_defocus else None
    r = orc.run_offline(fs, oc, seq, W.iters, workers=workers, mode=W.mode, tile_defocus=defocus,
                        want_tiles=False, want_stitched=False)
    return T * len(seq) * W.iters / r.wall_s, r.wall_s, T


def cpu_sample_desc(W: Workload, T: int, cores: int) -> str:
    return (f"{T} tile(s) (the FOV's first tile rows) x {W.leds} LEDs x {W.iters} iters {W.mode.upper()} "
            f"per step, oracle run_offline restatement, {cores} threads")


def repo_libs_loaded() -> list:
    """In-tree shared libraries mapped into this process (evidence of which code ran)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {l.split()[-1] for l in f if l.rstrip().endswith(".so")}
    except OSError:
        return []
    return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT + os.sep))


def run_reference(args, W: Workload, rank, world):
    """The reference's multithreaded CPU path (oracle port of run_offline,
    parallel.cpp:155-196) on rank 0; other ranks exit without work."""
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    rates = []
    for k in range(args.warmup + args.steps):
        rate, wall, T = cpu_sample(W, cores)
        if k >= args.warmup:
            rates.append(rate)
    v = float(np.mean(rates))
    line = {"impl": "reference", "metric": W.metric, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * T * W.leds * W.iters / v,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_block(W, world, args.scaling),
            "parallelism": f"cpu x{cores} threads (tile pool, parallel.cpp:126-140)",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": cpu_sample_desc(W, T, cores)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "full_recon_s": W.updates / v, "full_recon_s_note": "extrapolated from the sampled rate",
            "repo_native_libs_loaded": repo_libs_loaded()}
    assert "paper_2203_02507_b200" not in sys.modules, "the reference arm must not import the product"
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg
def run_b200(args, W: Workload, rank, world):
    import torch
    import torch.distributed as dist
    import paper_2203_02507_b200 as fpm
    from paper_2203_02507_b200.distributed import (PeerMosaic, allreduce_sum, band_layout, broadcast_from_rank0,
                                                   shard_request, stitch_band)

    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # collectives: NCCL on the device (the product setup); --dist-backend gloo runs the same
    # multi-rank path with host-side collectives, e.g. several ranks sharing one GPU for a
    # functional check of the strong-scaled step (not a measurement)
    nccl = args.dist_backend == "nccl"
    cdev = dev if nccl else torch.device("cpu")
    if world > 1:
        if nccl:
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    cfg = workload_cfg(W)
    seq, xy_all, of_all, defocus_all = geometry(W, cfg)
    L = len(seq)
    full = fpm.Request(cfg, W.iters, xy_all, of_all, np.arange(L, dtype=np.int32), 0, L, W.fov, W.fov, mode=W.mode,
                       tile_defocus_um=defocus_all)
    strong = args.scaling == "strong"
    multi = strong and world > 1  # one FOV over several GPUs: the mosaic bands meet in rank 0's buffer
    shards = [shard_request(full, r, world) for r in range(world)] if strong else None
    me = shards[rank] if strong else shard_request(full, 0, 1)
    T, H = len(me.tiles), me.y_hi - me.y_lo
    eng = fpm.Engine(local)
    plan = fpm.Plan(me.request, eng)
    info = plan.info
    abut = bool(info["tiles_abut"])
    lay = band_layout(cfg, xy_all, me.tile_lo, me.tile_hi)

    # device-resident synthetic stack (this rank's band of LR rows), frame k = LED seq[k]
    g = torch.Generator(device=dev)
    g.manual_seed(1 + rank)
    frames = torch.empty((L, H, W.fov), dtype=torch.uint16, device=dev)
    for k in range(L):  # per frame, to bound the int32 temporary
        frames[k] = torch.randint(0, 52429, (H, W.fov), dtype=torch.int32, device=dev, generator=g).to(torch.uint16)
    N = 4 * W.n
    resid = torch.empty((T, W.iters), dtype=torch.float64, device=dev)
    hr = None if abut else torch.empty((T, N, N, 2), dtype=torch.float32, device=dev)
    # the FOV's mosaic (stitch_mosaic, part of run_offline's wall clock, parallel.cpp:183): on rank 0,
    # written by every rank over NVLink (CUDA IPC) in the strong-scaled run
    mosaic = (torch.empty((lay.rows, lay.cols, 2), dtype=torch.float32, device=dev)
              if (rank == 0 or not multi) else None)
    peer = PeerMosaic(eng, rank, mosaic.data_ptr() if mosaic is not None else None,
                      broadcast_from_rank0(dev if nccl else None)) if multi else None
    mosaic_ptr = peer.ptr if multi else mosaic.data_ptr()
    band_ptr = mosaic_ptr + lay.row_lo * lay.cols * 8  # the band's top-left tile (abutting tiles)
    token = torch.zeros(1, dtype=torch.float32, device=cdev)
    combine = allreduce_sum(dev if nccl else None) if multi else None
    stream = torch.cuda.current_stream(dev)
    share = world if strong else 1  # ranks sharing one FOV's stack
    flush = l2_flush_needed(W, share)
    scrub = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev) if flush else None

    def step():
        if abut:  # canvas_to_field writes the HR fields straight into the (peer) mosaic
            plan.execute_mosaic(frames.data_ptr(), W.fov, band_ptr, lay.cols, resid.data_ptr(), None,
                                stream.cuda_stream)
        else:
            plan.execute(frames.data_ptr(), W.fov, hr.data_ptr(), resid.data_ptr(), None, stream.cuda_stream)
            stitch_band(eng, cfg, xy_all, me.tile_lo, me.tile_hi, hr.data_ptr(), mosaic_ptr, lay.cols, combine,
                        stream.cuda_stream)
        if multi:  # every band of rank 0's mosaic is written once every rank's kernels are past this point
            if not nccl:
                stream.synchronize()
            dist.all_reduce(token)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.phase_times(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        if flush:
            for e0, e1 in evs:
                scrub.zero_()  # evict the (L2-sized) inputs between timed steps
                e0.record(stream)
                step()
                e1.record(stream)
        else:
            evs[0][0].record(stream)
            for _ in range(args.steps):
                step()
            evs[-1][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = (sum(e0.elapsed_time(e1) for e0, e1 in evs) if flush else evs[0][0].elapsed_time(evs[-1][1])) / args.steps
    (ms_init, ms_loop, ms_fin), nexec = plan.phase_times(reset=True)
    assert nexec == args.steps, nexec
    ms_loop, ms_init, ms_fin = ms_loop / nexec, ms_init / nexec, ms_fin / nexec
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ok = bool(torch.isfinite(resid).all().item())
    units = W.updates * (1 if strong else world)  # weak: every rank ran the full workload
    value = units / (ms / 1000.0)

    e2e = None
    if not args.no_e2e:
        if multi:
            e2e = e2e_strong(args, W, me, plan, lay, band_ptr, abut, mosaic, rank, world, dev, cdev)
        else:  # one GPU (or weak scaling: every rank its own FOV) through the host-buffer C-ABI call
            e2e = e2e_leg(args, W, cfg, seq, xy_all, of_all, defocus_all, eng, world, cdev)

    out = None
    if rank == 0:
        flops_launch = info["fft_flops_per_update"] * info["updates"]
        bytes_launch = info["hbm_bytes_per_update"] * info["updates"]
        props = torch.cuda.get_device_properties(dev)
        sm_count = props.multi_processor_count
        pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
        peaks = json.load(open(pk)) if os.path.exists(pk) else {}
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        fp32_peak = sm_count * 128 * 2 * sm_max * 1e6 / 1e12  # TFLOP/s, FFMA lanes x 2 at max clock
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        achieved = flops_launch / (ms_loop / 1000.0) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "loop_kernel_dram_bytes.json")
        if os.path.exists(tp) and W.key == 3 and not multi:
            try:
                traffic = json.load(open(tp)).get("dram_bytes_per_launch_config3")
            except (OSError, ValueError):
                traffic = None
        cl = info["loop_ctas"] // max(info["num_tiles"], 1)
        if cl > 1:
            kernel = (f"fpm_loop_cluster (fused per-LED update, one tile over a {cl}-CTA cluster, DSMEM column "
                      "slabs, warp FFTs over the pupil box)")
        elif W.n == 64:
            kernel = (f"fpm_loop64 (fused per-LED update, {info['loop_threads']}-thread tile, "
                      "persistent over iters x LEDs)")
        else:
            kernel = "fpm_loop_box (fused per-LED update, warp FFTs over the pupil box)"
        # single-tile workloads cannot fill the GPU: also quote the roofline of the SMs they occupy
        sms_used = min(sm_count, info["loop_ctas"])
        out = {"metric": W.metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": args.scaling, "vs_baseline": None, "dtype": "f32 (complex64)", "data": "synthetic",
               "config": config_block(W, world, args.scaling),
               "parallelism": (f"tile-row bands x{world}, each rank writing its band of rank 0's mosaic over "
                               "NVLink (CUDA IPC peer pointer)" if multi else
                               f"one independent FOV per GPU x{world}" if world > 1 else "tiles->CTAs, 1 GPU"),
               "step": ("pupils + init_canvas + LED loop + canvas_to_field written straight into the FOV mosaic "
                        "(tiles abut: stitch_mosaic is a placement)" if abut else
                        "pupils + init_canvas + LED loop + canvas_to_field + Eq. (1) stitch_mosaic"),
               "full_recon_s": ms / 1000.0,
               "roofline": {"kernel": kernel, "bound": "fp32", "achieved": achieved, "peak": fp32_peak,
                            "unit": "TFLOP/s", "frac": achieved / fp32_peak, "traffic": traffic,
                            "peak_source": f"nominal FP32: {sm_count} SMs x 128 FMA lanes x 2 x {sm_max:.0f} MHz "
                                           "(MEASURED_PEAKS.json has no FP32 figure)",
                            "algorithmic_flops_per_launch": flops_launch,
                            "flops_per_update": info["fft_flops_per_update"],
                            "hbm_view": {"algorithmic_bytes_per_launch": bytes_launch,
                                         "achieved_gbs": bytes_launch / (ms_loop / 1000.0) / 1e9,
                                         "peak_gbs": hbm_peak,
                                         "frac": bytes_launch / (ms_loop / 1000.0) / 1e9 / hbm_peak},
                            "sms_used": sms_used,
                            "frac_of_sms_used": achieved / (fp32_peak * sms_used / sm_count),
                            "loop_ms": ms_loop, "init_ms": ms_init, "finalize_ms": ms_fin,
                            "loop_share_of_step": ms_loop / ms,
                            "measured_on": "rank 0's band" if multi else "the whole FOV"},
               "clocks": clk.summary(),
               "gpu_launches": (info["launches_per_execute"] + (0 if abut else 3)) * args.steps,
               "residuals_finite": ok}
        if e2e is not None:
            out["e2e"] = e2e
        if not args.no_cpu:
            cores = os.cpu_count() or 1
            rate, wall, Tc = cpu_sample(W, cores)
            out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                                   "sample": cpu_sample_desc(W, Tc, cores) + f", {wall:.1f} s"}
        print(json.dumps(out), flush=True)
    if peer is not None:
        if world > 1:
            dist.barrier()  # no rank writes into rank 0's mosaic any more
        peer.close()
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def e2e_strong(args, W: Workload, me, plan, lay, band_ptr: int, abut: bool, mosaic, rank: int, world: int, dev,
               cdev):
    """BASELINE config 4 end to end: every rank uploads its band of the LR stack
    from pinned host memory, reconstructs it and writes its band of rank 0's
    mosaic over NVLink; rank 0 copies the mosaic and every rank its residuals
    back to the host. Wall clock per step, max over ranks."""
    import torch
    import torch.distributed as dist
    if not abut:
        return None  # BASELINE configs abut (overlap 0); the overlapping mosaic path is covered by the GPU tests
    L, H, T = len(me.request.seq_frame), me.y_hi - me.y_lo, len(me.tiles)
    g = torch.Generator()
    g.manual_seed(1 + rank)
    host = torch.empty((L, H, W.fov), dtype=torch.uint16).pin_memory()
    for k in range(L):
        host[k] = torch.randint(0, 52429, (H, W.fov), dtype=torch.int32, generator=g).to(torch.uint16)
    frames = torch.empty((L, H, W.fov), dtype=torch.uint16, device=dev)
    resid = torch.empty((T, W.iters), dtype=torch.float64, device=dev)
    res_host = torch.empty((T, W.iters), dtype=torch.float64).pin_memory()
    mos_host = torch.empty(tuple(mosaic.shape), dtype=torch.float32).pin_memory() if rank == 0 else None
    token = torch.zeros(1, dtype=torch.float32, device=cdev)
    stream = torch.cuda.current_stream(dev)

    def step():
        frames.copy_(host, non_blocking=True)
        plan.execute_mosaic(frames.data_ptr(), W.fov, band_ptr, lay.cols, resid.data_ptr(), None, stream.cuda_stream)
        res_host.copy_(resid, non_blocking=True)
        if cdev.type == "cpu":
            stream.synchronize()
        dist.all_reduce(token)
        if rank == 0:
            mos_host.copy_(mosaic, non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(max(1, args.warmup)):
        step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    wall = (time.perf_counter() - t0) / args.steps
    t = torch.tensor([wall], dtype=torch.float64, device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall = float(t.item())
    h2d = torch.tensor([host.numel() * 2], dtype=torch.float64, device=cdev)
    dist.all_reduce(h2d)
    d2h = W.tiles * W.iters * 8 + lay.rows * lay.cols * 8
    return {"value": W.updates / wall, "unit": UNIT, "ms_per_step": wall * 1000.0,
            "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": int(d2h),
            "path": f"{world} ranks: pinned host band of the LR stack -> H2D -> plan execute_mosaic writing rank "
                    "0's mosaic over NVLink -> mosaic (rank 0) and residuals (every rank) back to pinned host "
                    "memory; one FOV per step, wall clock, max over ranks"}


def e2e_leg(args, W: Workload, cfg, seq, xy, of, defocus, eng, world: int = 1, cdev=None):
    """Same metric through the reference-facing host-buffer call (fpmgpu_reconstruct_tiles):
    pinned host LR stack -> H2D -> reconstruct -> D2H of HR tiles + residuals, every step.
    With N ranks (weak scaling) every rank times its own FOV; the slowest rank's wall
    time over the steps counts, and value = all ranks' updates / that time."""
    import ctypes as C

    import torch
    import paper_2203_02507_b200 as fpm
    from paper_2203_02507_b200._lib import check, lib
    L = len(seq)
    g = torch.Generator()
    g.manual_seed(1)
    host = torch.empty((L, W.fov, W.fov), dtype=torch.uint16).pin_memory()
    for k in range(L):
        host[k] = torch.randint(0, 52429, (W.fov, W.fov), dtype=torch.int32, generator=g).to(torch.uint16)
    req = fpm.Request(cfg, W.iters, xy, of, np.arange(L, dtype=np.int32), 0, L, W.fov, W.fov, mode=W.mode,
                      tile_defocus_um=defocus)
    N = 4 * W.n
    # two result buffers: consecutive requests are in flight together in the pipelined loop
    hr_host = [torch.empty((len(xy), N, N, 2), dtype=torch.float32).pin_memory() for _ in range(2)]
    res_host = [torch.empty((len(xy), W.iters), dtype=torch.float64).pin_memory() for _ in range(2)]
    r, keep = req.c()
    frames_ptr = host.data_ptr()

    def call():  # the synchronous reference-facing call
        check(lib().fpmgpu_reconstruct_tiles(eng.handle, C.byref(r), frames_ptr, W.fov, hr_host[0].data_ptr(),
                                             res_host[0].data_ptr(), None, None))

    def submit(k):  # the same call split: request k's upload runs under request k-1's reconstruction
        t = C.c_longlong()
        check(lib().fpmgpu_reconstruct_tiles_async(eng.handle, C.byref(r), frames_ptr, W.fov,
                                                   hr_host[k & 1].data_ptr(), res_host[k & 1].data_ptr(), None,
                                                   C.byref(t)))
        return t.value

    def wait(t):
        check(lib().fpmgpu_wait(eng.handle, C.c_longlong(t), None))

    def pipelined(steps):
        pending = []
        for k in range(steps):
            pending.append(submit(k))
            if len(pending) == 2:
                wait(pending.pop(0))
        for t in pending:
            wait(t)

    def timed(fn):
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        t0 = time.perf_counter()
        fn()
        wall = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([wall], dtype=torch.float64,
                             device=cdev if cdev is not None else torch.device("cuda", torch.cuda.current_device()))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall = float(t.item())
        return wall

    # each mode warmed up right before it is timed (they cut the tiles into different band counts)
    for _ in range(max(1, args.warmup)):
        call()
    wall_sync = timed(lambda: [call() for _ in range(args.steps)])
    pipelined(max(2, args.warmup))  # builds both slots' plans
    wall = timed(lambda: pipelined(args.steps))
    del keep
    ranks = f", {world} ranks, max over ranks" if world > 1 else ""
    h2d = int(host.numel() * 2) * world
    d2h = int(hr_host[0].numel() * 4 + res_host[0].numel() * 8) * world
    return {"value": world * W.updates / wall, "unit": UNIT, "ms_per_step": wall * 1000.0,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "fpmgpu_reconstruct_tiles_async + fpmgpu_wait (host buffers, pinned): K requests back to "
                    "back, request k+1's LR upload overlapping request k's reconstruction, every request's "
                    "H2D and HR/residual D2H inside the wall-clock region" + ranks,
            "sync": {"value": world * W.updates / wall_sync, "ms_per_step": wall_sync * 1000.0,
                     "path": "fpmgpu_reconstruct_tiles, one synchronous call per step (latency of one "
                             "reconstruction incl. copies)" + ranks}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", type=int, choices=sorted(WORKLOADS), default=3)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", choices=["gs", "epry"], default=None,
                    help="override the workload's update rule (default: the BASELINE config's)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="collectives under torchrun (gloo: host-side, e.g. ranks sharing one GPU for a functional check)")
    args = ap.parse_args()
    if args.impl == "b200":
        args.warmup = max(args.warmup, 3)
    W = WORKLOADS[args.config]
    if args.mode:  # e.g. config 3 in GS mode: the reference's own update rule (EPRY is an extension)
        from dataclasses import replace
        W = replace(W, mode=args.mode)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference(args, W, rank, world)
    return run_b200(args, W, rank, world)


if __name__ == "__main__":
    sys.exit(main())
