"""Cases for the bounds-checked build (tests/test_gpu_checked.py): every kernel
family and host path of the product, small sizes. Run as a script it writes the
results to an .npz; the test runs it once with FPM_B200_LIB=check (device
asserts that trap on any out-of-range index, make check) in a subprocess and
compares with the production build in process.

    python tests/checked_cases.py out.npz
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2203_02507_b200 as fpm  # noqa: E402
from tests.helpers import dataset, gpu_cfg  # noqa: E402


def _env(env: dict):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    return old


def _restore(old: dict):
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _offline(env, cfg, fov, mode, iters, seed, defocus=None):
    old = _env({"FPM_B200_BANDS": "1", **env})
    try:
        fs, _, seq, _ = dataset(cfg, fov=fov, seed=seed, defocus_um=4.0 if cfg.tile_size > 64 else 0.0)
        specs = fpm.partition_tiles(fs.width(), fs.height(), cfg)
        dz = list(np.linspace(-6, 6, len(specs))) if defocus else None
        opt = fpm.RunOptions(iters=iters, mode=mode, tile_defocus_um=dz)
        r = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=True)
        out = {"tiles": r.tiles, "resid": np.array([m.pass_mean_residual for m in r.tile_metrics])}
        if r.stitched is not None:
            out["mosaic"] = r.stitched
        if r.pupils is not None:
            out["pupils"] = np.asarray(r.pupils)
        return out
    finally:
        _restore(old)


def cases():
    n64 = gpu_cfg(led_scan_rows=7, led_scan_cols=7, tile_overlap=8)
    n128 = fpm.OpticalConfig(tile_size=128, tile_overlap=0, upsample=4, led_scan_rows=5, led_scan_cols=5)
    n256 = fpm.OpticalConfig(tile_size=256, tile_overlap=0, upsample=4, led_scan_rows=3, led_scan_cols=3)
    return {
        # fpm_loop64, one CTA per tile and as the work queue; banded async host path
        "pair_ctas": lambda: _offline(dict(FPM_B200_QUAD="0", FPM_B200_QUEUE="0"), n64, 232, "epry", 2, 70, True),
        "pair_queue": lambda: _offline(dict(FPM_B200_QUAD="0", FPM_B200_QUEUE="1"), n64, 232, "epry", 2, 71, True),
        "pair_gs_bands": lambda: _offline(dict(FPM_B200_QUAD="0", FPM_B200_BANDS="3"), n64, 232, "gs", 2, 72),
        # fpm_loop64q
        "quad_queue": lambda: _offline(dict(FPM_B200_QUAD="1", FPM_B200_QUEUE="1"), n64, 232, "epry", 2, 73, True),
        # fpm_loop_box / fpm_loop_cluster (st.async n = 128; n = 256 WarpFFT256, pruned and full)
        "box128": lambda: _offline(dict(FPM_B200_CLUSTER="1"), n128, 128, "epry", 2, 74),
        "cluster128": lambda: _offline(dict(FPM_B200_CLUSTER="8"), n128, 128, "epry", 2, 75),
        "cluster256_queue": lambda: _offline(dict(FPM_B200_CLUSTER="4", FPM_B200_QUEUE="1"), n256, 512, "epry", 2, 76,
                                             True),
        "cluster256_full": lambda: _offline(dict(FPM_B200_CLUSTER="4", FPM_B200_MID="0"), n256, 256, "gs", 2, 77),
        "box256": lambda: _offline(dict(FPM_B200_CLUSTER="1"), n256, 256, "epry", 1, 78),
    }


def pipelined_case():
    """The pipelined GS schedule (G > 1 slot groups) on one tile."""
    cfg = gpu_cfg(led_scan_rows=7, led_scan_cols=7)
    fs, _, seq, _ = dataset(cfg, seed=79)
    t = fpm.partition_tiles(64, 64, cfg)[0]
    r = fpm.pipelined_reconstruct_tile(fs, t, cfg, 2, seq, engine=fpm.Engine(0))
    return {"hr": r.hr, "resid": np.asarray(r.metrics.pass_mean_residual)}


def run_all() -> dict:
    out = {}
    for name, fn in cases().items():
        for k, v in fn().items():
            out[f"{name}/{k}"] = v
    for k, v in pipelined_case().items():
        out[f"pipelined/{k}"] = v
    return out


if __name__ == "__main__":
    res = run_all()
    np.savez(sys.argv[1], **res)
    print(f"checked cases: {len(res)} arrays, library {fpm._lib.LIB_PATH}")
