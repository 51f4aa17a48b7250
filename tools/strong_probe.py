"""One rank's share of a strong-scaled run (BASELINE config 4/5 over G GPUs), on
one GPU: the rank-0 tile-row band of shard_request(full, 0, G), device-resident,
timed with CUDA events. Prints one line per G. Used to pick the kernel for
small per-GPU tile counts (FPM_B200_CLUSTER etc. in the environment).

    python tools/strong_probe.py [--config 3|5] [--gpus 1 2 4 8]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2203_02507_b200 as fpm
    from paper_2203_02507_b200.distributed import shard_request

    W = bench.WORKLOADS[a.config]
    cfg = bench.workload_cfg(W)
    seq, xy, of, defocus = bench.geometry(W, cfg)
    L = len(seq)
    full = fpm.Request(cfg, W.iters, xy, of, np.arange(L, dtype=np.int32), 0, L, W.fov, W.fov, mode=W.mode,
                       tile_defocus_um=defocus)
    dev = torch.device("cuda", 0)
    eng = fpm.Engine(0)
    for G in a.gpus:
        me = shard_request(full, 0, G)
        T, H = len(me.tiles), me.y_hi - me.y_lo
        plan = fpm.Plan(me.request, eng)
        frames = torch.randint(0, 52429, (L, H, W.fov), dtype=torch.int32, device=dev).to(torch.uint16)
        N = 4 * W.n
        hr = torch.empty((T, N, N, 2), dtype=torch.float32, device=dev)
        resid = torch.empty((T, W.iters), dtype=torch.float64, device=dev)
        s = torch.cuda.current_stream(dev)
        plan.execute(frames.data_ptr(), W.fov, hr.data_ptr(), resid.data_ptr(), None, s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.steps):
            plan.execute(frames.data_ptr(), W.fov, hr.data_ptr(), resid.data_ptr(), None, s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        upd = T * L * W.iters
        print(f"config {a.config} G={G}: {T} tiles/GPU, {ms:.2f} ms per step, {upd / ms / 1e3:.3f} M updates/s per GPU, "
              f"{G * upd / ms / 1e3:.3f} M/s for {G} GPUs (if linear)", flush=True)
        del frames, hr, resid, plan


if __name__ == "__main__":
    main()
