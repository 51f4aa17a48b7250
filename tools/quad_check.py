"""Quad-lattice kernel (FPM_B200_QUAD=1) against the pair lattice and the oracle
on a small EPRY batch; prints the max relative differences."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2203_02507_b200 as fpm  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from tests.helpers import amp_phase_rel, dataset, gpu_cfg, orc_cfg, rel_l2  # noqa: E402

for mode in ("gs", "epry"):
    cfg = gpu_cfg(led_scan_rows=7, led_scan_cols=7, tile_overlap=8)
    fs, ofs, seq, _ = dataset(cfg, fov=176, seed=35)
    specs = fpm.partition_tiles(fs.width(), fs.height(), cfg)
    dz = list(np.linspace(-6, 6, len(specs)))
    opt = fpm.RunOptions(iters=3, mode=mode, tile_defocus_um=dz)
    os.environ["FPM_B200_QUAD"] = "0"
    a = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    for q in ("0", "1"):
        os.environ["FPM_B200_QUEUE"] = q
        os.environ["FPM_B200_QUAD"] = "1"
        b = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
        d = max(rel_l2(b.tiles[i], a.tiles[i]) for i in range(len(specs)))
        ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), 3, seq, tile_index=2, mode=mode, tile_defocus=dz[2])
        amp, ph = amp_phase_rel(b.tiles[2], ref.hr)
        rr = np.max(np.abs(np.array(b.tile_metrics[2].pass_mean_residual) / ref.residuals - 1))
        print(f"{mode} queue={q}: quad vs pair max rel-L2 {d:.2e}; tile 2 vs oracle amp {amp:.2e} phase {ph:.2e} "
              f"resid {rr:.2e}", flush=True)
    os.environ.pop("FPM_B200_QUEUE")
