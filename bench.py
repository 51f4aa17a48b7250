"""Benchmark: LED-updates/s of the FPM reconstruction (default: BASELINE config 3).

Default workload (config 3, N=1): 2048x2048 sensor, 32x32 tiles of 64x64 LR
px (overlap 0), 15x15 LEDs (spiral order), 10 iterations EPRY, per-tile
illumination k-vectors and per-tile defocus pupils (uniform +-10 um, seed 7);
synthetic u16 LR stack (uniform [0, 52428], seed 1: the cost is
data-independent). One step = one full reconstruction (pupils + init_canvas +
LED loop + canvas_to_field) of every tile. Under torchrun (N > 1) the
default is weak scaling: tiles are independent units, so every
rank reconstructs its own full config-3 FOV (its own synthetic stack) with no
collective in the step, and `value` = all ranks' updates / the slowest rank's
time. `--scaling strong` runs BASELINE config 4 instead: one FOV sharded in
contiguous tile-row bands over the ranks, each holding only its band of the
stack, the HR tiles gathered to rank 0 by NCCL (the only inter-GPU step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config 3|1|2|5] [--scaling weak|strong] [--no-e2e] [--no-cpu]

`--config` 1/2/5 measure the other BASELINE shapes (single 64 px tile GS;
single 128 px tile EPRY; 4096x4096 sensor of 256 px tiles, 21x21 LEDs).
`--impl reference` times the CPU oracle's restatement of the reference's
multithreaded run_offline (the reference itself cannot be built here: no
Eigen) on a bounded sample of the same workload, with every host thread.
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


def geometry(W: Workload, cfg):
    import paper_2203_02507_b200 as fpm
    seq = fpm.led_sequence("spiral", cfg)
    xy, _, _, of = fpm.partition_arrays(W.fov, W.fov, cfg, seq)
    defocus = np.random.default_rng(7).uniform(-10.0, 10.0, len(xy)) if W.per_tile_defocus else None
    return seq, xy, of, defocus


def l2_flush_needed(W: Workload, world: int) -> bool:
    return W.stack_bytes // max(world, 1) < 256 * 1024 * 1024


def config_block(W: Workload, world: int, extra=None):
    c = {"workload": f"{W.label}: {W.fov}x{W.fov} sensor, {W.tiles} tiles n={W.n} (N={4 * W.n}), "
                     f"{W.scan}x{W.scan} LEDs spiral, {W.iters} iters {W.mode.upper()}"
                     + (", per-tile k-vectors + defocus pupils" if W.per_tile_defocus else ""),
         "baseline_config": W.key, "fov": W.fov, "tile_side": W.n, "canvas_side": 4 * W.n, "leds": W.leds,
         "iters": W.iters, "mode": W.mode, "tiles": W.tiles, "updates_per_step": W.updates,
         "l2_policy": ("L2 flushed (256 MiB write) between timed steps; per-step CUDA events"
                       if l2_flush_needed(W, world) else
                       f"inputs larger than L2 (LR stack {W.stack_bytes / 2**30:.2f} GiB)")}
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
def cpu_sample(W: Workload, cfg_gpu, seq, workers: int):
    """Oracle run_offline on the first tile row of the workload (fov x n crop), one
    iteration, same mode and per-tile defocus; returns (updates/s, wall, tiles)."""
    from oracle import oracle as orc
    oc = orc.Optics(**{f: getattr(cfg_gpu, f) for f in orc.Optics.__dataclass_fields__})
    H = W.n
    rng = np.random.default_rng(1)
    imgs = rng.integers(0, 52429, (len(seq), H, W.fov), dtype=np.uint16)
    fs = orc.FrameStack(imgs, [tuple(l) for l in seq])
    T = W.fov // W.n
    if W.mode != "gs":  # the pipelined path (workers > tiles, parallel.cpp:166) is GS-only
        workers = min(workers, T)
    defocus = np.random.default_rng(7).uniform(-10.0, 10.0, T) if W.per_tile_defocus else None
    r = orc.run_offline(fs, oc, seq, 1, workers=workers, mode=W.mode, tile_defocus=defocus,
                        want_tiles=False, want_stitched=False)
    return T * len(seq) / r.wall_s, r.wall_s, T


def cpu_sample_desc(W: Workload, T: int, cores: int) -> str:
    return (f"{T} tile(s) (first tile row) x {W.leds} LEDs x 1 iter {W.mode.upper()} per step, oracle "
            f"run_offline restatement, {cores} threads")


def run_reference(args, W: Workload, rank, world):
    if rank != 0:
        return 0
    cfg = workload_cfg(W)
    seq, _, _, _ = geometry(W, cfg)
    cores = os.cpu_count() or 1
    rates = []
    for k in range(args.warmup + args.steps):
        rate, wall, T = cpu_sample(W, cfg, seq, cores)
        if k >= args.warmup:
            rates.append(rate)
    v = float(np.mean(rates))
    line = {"impl": "reference", "metric": W.metric, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * T * len(seq) / v,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_block(W, 1, {"parallelism": f"cpu x{cores} threads (tile pool, parallel.cpp:126-140)"}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": cpu_sample_desc(W, T, cores)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "full_recon_s_extrapolated": W.updates / v}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg
def run_b200(args, W: Workload, rank, world):
    import torch
    import torch.distributed as dist
    import paper_2203_02507_b200 as fpm
    from paper_2203_02507_b200.distributed import gather_tiles, shard_request

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = workload_cfg(W)
    seq, xy_all, of_all, defocus_all = geometry(W, cfg)
    L = len(seq)
    full = fpm.Request(cfg, W.iters, xy_all, of_all, np.arange(L, dtype=np.int32), 0, L, W.fov, W.fov, mode=W.mode,
                       tile_defocus_um=defocus_all)
    strong = args.scaling == "strong" and world > 1
    shards = [shard_request(full, r, world) for r in range(world)] if strong else None
    me = shards[rank] if strong else shard_request(full, 0, 1)
    T, H = len(me.tiles), me.y_hi - me.y_lo
    eng = fpm.Engine(local)
    plan = fpm.Plan(me.request, eng)
    info = plan.info

    # device-resident synthetic stack (this rank's band of LR rows), frame k = LED seq[k]
    g = torch.Generator(device=dev)
    g.manual_seed(1 + rank)
    frames = torch.empty((L, H, W.fov), dtype=torch.uint16, device=dev)
    for k in range(L):  # per frame, to bound the int32 temporary
        frames[k] = torch.randint(0, 52429, (H, W.fov), dtype=torch.int32, device=dev, generator=g).to(torch.uint16)
    N = 4 * W.n
    hr = torch.empty((T, N, N, 2), dtype=torch.float32, device=dev)
    resid = torch.empty((T, W.iters), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    mosaic_tiles = torch.empty((len(xy_all), N, N, 2), dtype=torch.float32, device=dev) if (
        strong and rank == 0) else None
    share = world if strong else 1  # ranks sharing one FOV's stack
    flush = l2_flush_needed(W, share)
    scrub = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev) if flush else None

    def step():
        plan.execute(frames.data_ptr(), W.fov, hr.data_ptr(), resid.data_ptr(), None, stream.cuda_stream)
        if strong:  # the only inter-GPU step: HR tiles gathered to rank 0 (NCCL send/recv)
            gather_tiles(hr, shards, rank, mosaic_tiles.shape if rank == 0 else None, out=mosaic_tiles)

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
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ok = bool(torch.isfinite(resid).all().item())
    units = W.updates * (1 if strong else world)  # weak: every rank ran the full workload
    value = units / (ms / 1000.0)

    # e2e through the host-buffer C-ABI call: every rank (weak scaling: each its own FOV)
    e2e = None
    if not args.no_e2e and not strong:
        e2e = e2e_leg(args, W, cfg, seq, xy_all, of_all, defocus_all, eng, world)

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
        if os.path.exists(tp) and W.key == 3:
            try:
                traffic = json.load(open(tp)).get("dram_bytes_per_launch_config3")
            except (OSError, ValueError):
                traffic = None
        cl = info["loop_ctas"] // max(info["num_tiles"], 1)
        if cl > 1:
            kernel = (f"fpm_loop_cluster (fused per-LED update, one tile over a {cl}-CTA cluster, DSMEM column "
                      "slabs, warp FFTs over the pupil box)")
        elif W.n == 64:
            kernel = "fpm_loop64 (fused per-LED update, 128-thread pair lattice, persistent over iters x LEDs)"
        else:
            kernel = "fpm_loop_box (fused per-LED update, warp FFTs over the pupil box)"
        # single-tile workloads cannot fill the GPU: also quote the roofline of the SMs they occupy
        sms_used = min(sm_count, info["loop_ctas"])
        out = {"metric": W.metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "strong" if strong else "weak",
               "vs_baseline": None, "dtype": "f32 (complex64)", "data": "synthetic",
               "config": config_block(W, share, {
                   "parallelism": (f"tile-row bands x{world} + NCCL HR gather (config 4)" if strong else
                                   f"one independent FOV per GPU x{world}" if world > 1 else "tiles->CTAs, 1 GPU"),
                   "updates_per_step_all_ranks": units, "full_recon_s": ms / 1000.0}),
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
                            "loop_share_of_step": ms_loop / ms},
               "clocks": clk.summary(),
               "gpu_launches": info["launches_per_execute"] * args.steps,
               "residuals_finite": ok}
        if e2e is not None:
            out["e2e"] = e2e
        if world == 1 and not args.no_cpu:
            cores = os.cpu_count() or 1
            rate, wall, Tc = cpu_sample(W, cfg, seq, cores)
            out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                                   "sample": cpu_sample_desc(W, Tc, cores) + f", {wall:.1f} s"}
        print(json.dumps(out), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_leg(args, W: Workload, cfg, seq, xy, of, defocus, eng, world: int = 1):
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
            t = torch.tensor([wall], dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
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
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    W = WORKLOADS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference(args, W, rank, world)
    return run_b200(args, W, rank, world)


if __name__ == "__main__":
    sys.exit(main())
