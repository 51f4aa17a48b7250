"""Benchmark: LED-updates/s of the full-FOV FPM reconstruction (BASELINE config 3).

Workload (N=1): 2048x2048 sensor, 32x32 tiles of 64x64 LR px (overlap 0),
15x15 LEDs (spiral order), 10 iterations EPRY, per-tile illumination
k-vectors and per-tile defocus pupils (uniform +-10 um, seed 7); synthetic
u16 LR stack (uniform [0, 52428], seed 1: the cost is data-independent).
One step = one full reconstruction (pupils + init_canvas + LED loop +
canvas_to_field) of every tile. Under torchrun the tiles are sharded in
contiguous tile-row bands over the ranks (strong scaling of config 4); each
rank holds only its band of the stack, the HR bands are gathered to rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

`--impl reference` times the CPU oracle's restatement of the reference's
multithreaded run_offline (the reference itself cannot be built here: no
Eigen) on a bounded sample of the same workload, with every host thread.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FOV = 2048
SCAN = 15
ITERS = 10
MODE = "epry"
METRIC = "LED-updates/sec (full-FOV 2048x2048, 32x32 tiles of 64x64 LR, 15x15 LEDs, 10 iters EPRY)"
UNIT = "LED-updates/s"


def workload_cfg():
    import paper_2203_02507_b200 as fpm
    return fpm.OpticalConfig(tile_size=64, tile_overlap=0, upsample=4, led_scan_rows=SCAN, led_scan_cols=SCAN)


def geometry(cfg):
    import paper_2203_02507_b200 as fpm
    seq = fpm.led_sequence("spiral", cfg)
    xy, _, _, of = fpm.partition_arrays(FOV, FOV, cfg, seq)
    defocus = np.random.default_rng(7).uniform(-10.0, 10.0, len(xy))
    return seq, xy, of, defocus


def config_block(extra=None):
    c = {"workload": "BASELINE config 3/4: full FOV 2048x2048, 32x32 tiles n=64 (N=256), 15x15 LEDs spiral, "
                     "10 iters EPRY, per-tile k-vectors + defocus pupils",
         "fov": FOV, "tile_side": 64, "canvas_side": 256, "leds": SCAN * SCAN, "iters": ITERS, "mode": MODE,
         "tiles": 1024, "updates_per_step": 1024 * SCAN * SCAN * ITERS,
         "l2_policy": "inputs larger than L2 (LR stack 1.76 GiB, canvases 512 MiB per step)"}
    if extra:
        c.update(extra)
    return c


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
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
def cpu_sample(cfg_gpu, seq, tile_rows: int, iters: int, workers: int):
    """Oracle run_offline on the first `tile_rows` tile rows (2048 x 64*rows crop) of the
    workload, EPRY, per-tile defocus; returns (updates/s, wall, tiles)."""
    from oracle import oracle as orc
    oc = orc.Optics(**{f: getattr(cfg_gpu, f) for f in orc.Optics.__dataclass_fields__})
    H = 64 * tile_rows
    rng = np.random.default_rng(1)
    imgs = rng.integers(0, 52429, (len(seq), H, FOV), dtype=np.uint16)
    fs = orc.FrameStack(imgs, [tuple(l) for l in seq])
    T = (FOV // 64) * tile_rows
    defocus = np.random.default_rng(7).uniform(-10.0, 10.0, T)
    r = orc.run_offline(fs, oc, seq, iters, workers=workers, mode=MODE, tile_defocus=defocus,
                        want_tiles=False, want_stitched=False)
    upd = T * len(seq) * iters
    return upd / r.wall_s, r.wall_s, T


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cfg = workload_cfg()
    seq, _, _, _ = geometry(cfg)
    cores = os.cpu_count() or 1
    # each step: one tile row (32 tiles) x 1 iteration over 225 LEDs with every host thread
    rates = []
    for k in range(args.warmup + args.steps):
        rate, wall, T = cpu_sample(cfg, seq, 1, 1, cores)
        if k >= args.warmup:
            rates.append(rate)
    v = float(np.mean(rates))
    sample = f"{T} tiles (first tile row) x 225 LEDs x 1 iter EPRY per step, oracle run_offline, {cores} threads"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * T * len(seq) / v,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block({"parallelism": f"cpu x{cores} threads (tile pool, parallel.cpp:126-140)"}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "full_fov_recon_s_extrapolated": 1024 * 225 * ITERS / v}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg
def run_b200(args, rank, world):
    import torch
    import torch.distributed as dist
    import paper_2203_02507_b200 as fpm

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2203_02507_b200.distributed import gather_tiles, shard_request

    cfg = workload_cfg()
    seq, xy_all, of_all, defocus_all = geometry(cfg)
    L = len(seq)
    full = fpm.Request(cfg, ITERS, xy_all, of_all, np.arange(L, dtype=np.int32), 0, L, FOV, FOV, mode=MODE,
                       tile_defocus_um=defocus_all)
    shards = [shard_request(full, r, world) for r in range(world)]
    me = shards[rank]
    T, H = len(me.tiles), me.y_hi - me.y_lo
    eng = fpm.Engine(local)
    plan = fpm.Plan(me.request, eng)
    info = plan.info

    # device-resident synthetic stack (this rank's band of LR rows), frame k = LED seq[k]
    g = torch.Generator(device=dev)
    g.manual_seed(1 + rank)
    frames = torch.randint(0, 52429, (L, H, FOV), dtype=torch.int32, device=dev, generator=g).to(torch.uint16)
    N = 256
    hr = torch.empty((T, N, N, 2), dtype=torch.float32, device=dev)
    resid = torch.empty((T, ITERS), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    mosaic_tiles = torch.empty((len(xy_all), N, N, 2), dtype=torch.float32, device=dev) if (
        world > 1 and rank == 0) else None

    def step():
        plan.execute(frames.data_ptr(), FOV, hr.data_ptr(), resid.data_ptr(), None, stream.cuda_stream)
        if world > 1:  # the only inter-GPU step: HR tiles gathered to rank 0 (NCCL send/recv)
            gather_tiles(hr, shards, rank, mosaic_tiles.shape if rank == 0 else None, out=mosaic_tiles)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.phase_times(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    (ms_init, ms_loop, ms_fin), nexec = plan.phase_times(reset=True)
    assert nexec == args.steps, nexec
    ms_loop /= nexec
    ms_init /= nexec
    ms_fin /= nexec
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ok = bool(torch.isfinite(resid).all().item())

    total_updates = 1024 * L * ITERS
    value = total_updates / (ms / 1000.0)

    out = None
    if rank == 0:
        # roofline of the dominant kernel (the fused LED loop), per launch
        flops_launch = info["fft_flops_per_update"] * info["updates"]
        bytes_launch = info["hbm_bytes_per_update"] * info["updates"]
        props = torch.cuda.get_device_properties(dev)
        sm_count = props.multi_processor_count
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        fp32_peak = sm_count * 128 * 2 * sm_max * 1e6 / 1e12  # TFLOP/s, FFMA lanes x 2 at max clock
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        achieved = flops_launch / (ms_loop / 1000.0) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "loop_kernel_dram_bytes.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get("dram_bytes_per_launch_config3")
            except Exception:
                traffic = None
        clocks = clk.summary()
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f32 (complex64)", "data": "synthetic",
               "config": config_block({"parallelism": f"tile-shard x{world}" if world > 1 else "tiles->CTAs, 1 GPU",
                                       "full_fov_recon_s": ms / 1000.0}),
               "roofline": {"kernel": "fpm_loop64 (fused per-LED update, persistent over iters x LEDs)",
                            "bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                            "frac": achieved / fp32_peak, "traffic": traffic,
                            "peak_source": f"nominal FP32: {sm_count} SMs x 128 FMA lanes x 2 x {sm_max:.0f} MHz "
                                           "(MEASURED_PEAKS.json has no FP32 figure)",
                            "algorithmic_flops_per_launch": flops_launch,
                            "flops_per_update": info["fft_flops_per_update"],
                            "hbm_view": {"algorithmic_bytes_per_launch": bytes_launch,
                                         "achieved_gbs": bytes_launch / (ms_loop / 1000.0) / 1e9,
                                         "peak_gbs": hbm_peak, "frac": bytes_launch / (ms_loop / 1000.0) / 1e9 / hbm_peak},
                            "loop_ms": ms_loop, "init_ms": ms_init, "finalize_ms": ms_fin,
                            "loop_share_of_step": ms_loop / ms},
               "clocks": clocks,
               "gpu_launches": info["launches_per_execute"] * args.steps,
               "residuals_finite": ok}
    if not args.no_e2e and world == 1:
        out["e2e"] = e2e_leg(args, cfg, seq, xy_all, of_all, defocus_all, eng)
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        rate, wall, Tc = cpu_sample(cfg, seq, 1, 1, cores)
        out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                               "sample": f"{Tc} tiles (first tile row) x 225 LEDs x 1 iter EPRY, oracle "
                                         f"run_offline restatement, {cores} threads, {wall:.1f} s"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_leg(args, cfg, seq, xy, of, defocus, eng):
    """Same metric through the reference-facing host-buffer call (fpmgpu_reconstruct_tiles):
    pinned host LR stack -> H2D -> reconstruct -> D2H of HR tiles + residuals, every step."""
    import torch
    import paper_2203_02507_b200 as fpm
    L = len(seq)
    g = torch.Generator()
    g.manual_seed(1)
    host = torch.randint(0, 52429, (L, FOV, FOV), dtype=torch.int32, generator=g).to(torch.uint16).pin_memory()
    frames = fpm.FrameSet(host.numpy(), [tuple(l) for l in seq])
    req = fpm.Request(cfg, ITERS, xy, of, np.arange(L, dtype=np.int32), 0, L, FOV, FOV, mode=MODE,
                      tile_defocus_um=defocus)
    hr_host = torch.empty((len(xy), 256, 256, 2), dtype=torch.float32).pin_memory()
    res_host = torch.empty((len(xy), ITERS), dtype=torch.float64).pin_memory()
    r, keep = req.c()
    import ctypes as C
    from paper_2203_02507_b200._lib import check, lib

    def call():
        check(lib().fpmgpu_reconstruct_tiles(eng.handle, C.byref(r), frames.images.ctypes.data, FOV,
                                             hr_host.data_ptr(), res_host.data_ptr(), None, None))

    for _ in range(max(1, args.warmup)):
        call()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        call()
    wall = (time.perf_counter() - t0) / args.steps
    del keep
    return {"value": 1024 * L * ITERS / wall, "unit": UNIT, "ms_per_step": wall * 1000.0,
            "h2d_bytes_per_step": int(host.numel() * 2), "d2h_bytes_per_step": int(hr_host.numel() * 4 + res_host.numel() * 8),
            "path": "fpmgpu_reconstruct_tiles (host buffers, pinned), wall clock around the synchronous call"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world)


if __name__ == "__main__":
    sys.exit(main())
