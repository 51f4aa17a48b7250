"""Small reconstructions that drive each hand-synchronised kernel path, for
compute-sanitizer (racecheck / synccheck / memcheck) runs on the GPU box:

  compute-sanitizer --tool racecheck python tools/sanitize_case.py loop64_queue

Cases (each a few hundred updates so the instrumented run stays short):
  loop64_queue   fpm_loop64, persistent work queue forced (acquire/release item
                 protocol, TMA staging + cp.async EPRY staging behind proxy fences)
  loop64         fpm_loop64, one CTA per tile
  cluster128     fpm_loop_cluster n = 128 (st.async slab exchange + mbarriers)
  cluster256     fpm_loop_cluster n = 256, 4-CTA clusters, cluster work queue
  host_banded    the banded async host path (fpmgpu_reconstruct_tiles_async, 4 bands)
  mosaic         device stitch (sums + assembly) and execute_mosaic
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2203_02507_b200 as fpm  # noqa: E402


def stack(n, scan, fov, seed=1):
    rng = np.random.default_rng(seed)
    cfg = fpm.OpticalConfig(tile_size=n, tile_overlap=0, upsample=4, led_scan_rows=scan, led_scan_cols=scan)
    seq = fpm.led_sequence("spiral", cfg)
    imgs = rng.integers(100, 40000, (len(seq), fov, fov), dtype=np.uint16)
    return cfg, fpm.FrameSet(imgs, [tuple(s) for s in seq]), seq


def main(case):
    if case in ("loop64_queue", "loop64"):
        os.environ["FPM_B200_QUEUE"] = "1" if case == "loop64_queue" else "0"
        os.environ["FPM_B200_BANDS"] = "1"
        cfg, fs, seq = stack(64, 5, 256)
        r = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=2, mode="epry",
                                                         tile_defocus_um=list(np.linspace(-5, 5, 16))), stitch=False)
    elif case == "cluster128":
        os.environ["FPM_B200_CLUSTER"] = "8"
        cfg, fs, seq = stack(128, 5, 128)
        r = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=2, mode="epry"), stitch=False)
    elif case == "cluster256":
        os.environ["FPM_B200_CLUSTER"] = "4"
        os.environ["FPM_B200_QUEUE"] = "1"
        os.environ["FPM_B200_BANDS"] = "1"
        cfg, fs, seq = stack(256, 3, 512)
        r = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=2, mode="epry", tile_defocus_um=[1.0, -2.0, 3.0, 0.0]),
                            stitch=False)
    elif case == "host_banded":
        os.environ["FPM_B200_BANDS"] = "4"
        cfg, fs, seq = stack(64, 3, 256)
        specs = fpm.partition_tiles(256, 256, cfg)
        req = fpm.make_request(fs, cfg, seq, specs, 2, mode="epry")
        pend = [fpm.reconstruct_request_async(req, fs) for _ in range(3)]
        outs = [p.wait() for p in pend]
        assert all(np.array_equal(o[0], outs[0][0]) for o in outs)
        r = None
    elif case == "mosaic":
        import torch
        cfg, fs, seq = stack(64, 3, 256)
        cfg.tile_overlap = 8
        specs = fpm.partition_tiles(256, 256, cfg)
        r = fpm.run_offline(fs, cfg, seq, fpm.RunOptions(iters=1))
        assert r.stitched is not None
        cfg0, fs0, seq0 = stack(64, 3, 256)
        specs0 = fpm.partition_tiles(256, 256, cfg0)
        plan = fpm.Plan(fpm.make_request(fs0, cfg0, seq0, specs0, 1), fpm.default_engine())
        dev = torch.device("cuda", 0)
        frames = torch.from_numpy(fs0.images).to(dev)
        mosaic = torch.empty((1024, 1024, 2), dtype=torch.float32, device=dev)
        res = torch.empty((16, 1), dtype=torch.float64, device=dev)
        plan.execute_mosaic(frames.data_ptr(), 256, mosaic.data_ptr(), 1024, res.data_ptr(), None,
                            torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    else:
        raise SystemExit(f"unknown case {case}")
    if r is not None:
        assert np.isfinite(r.tiles).all()
    print(f"{case}: ok")


if __name__ == "__main__":
    main(sys.argv[1])
