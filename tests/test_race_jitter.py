"""Race hunting without compute-sanitizer (closed on the GPU pool, see
profiles/r2/compute_sanitizer_refused.txt): FPM_B200_JITTER makes every warp
sleep a pseudo-random 0..jitter ns before each update and each work-queue
claim, reshuffling warp and CTA interleavings. Every hand-synchronised path
must then give the unperturbed run's bits, for several seeds:

* fpm_loop64 (pair lattice), one CTA per tile and as the work queue
  (acquire/release item protocol, TMA staging behind proxy fences, the EPRY
  cp.async staging of the scatter operands);
* fpm_loop64q (quad lattice), work queue;
* fpm_loop_cluster n = 128 (st.async slab exchange counted on mbarriers, relaxed
  cluster arrives) and n = 256 (DSMEM row exchange, cluster work queue);
* fpm_loop_box n = 128 (one CTA, shared-memory box rows).

The disjoint-disk contract these protect is recon.cpp:105-106."""
import numpy as np
import pytest

import paper_2203_02507_b200 as fpm
from tests.helpers import dataset, gpu_cfg

pytestmark = pytest.mark.gpu

CASES = {
    "pair_queue": (dict(FPM_B200_QUAD="0", FPM_B200_QUEUE="1"), 64, 7, 232, "epry", 3),
    "pair_ctas": (dict(FPM_B200_QUAD="0", FPM_B200_QUEUE="0"), 64, 7, 232, "epry", 3),
    "pair_gs_queue": (dict(FPM_B200_QUAD="0", FPM_B200_QUEUE="1"), 64, 7, 232, "gs", 3),
    "quad_queue": (dict(FPM_B200_QUAD="1", FPM_B200_QUEUE="1"), 64, 7, 232, "epry", 3),
    "cluster128": (dict(FPM_B200_CLUSTER="8"), 128, 5, 128, "epry", 2),
    "cluster256_queue": (dict(FPM_B200_CLUSTER="4", FPM_B200_QUEUE="1"), 256, 3, 512, "epry", 2),
    "box128": (dict(FPM_B200_CLUSTER="1"), 128, 5, 256, "epry", 2),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_jitter_leaves_bits_unchanged(monkeypatch, case):
    env, n, scan, fov, mode, iters = CASES[case]
    monkeypatch.setenv("FPM_B200_BANDS", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = (gpu_cfg(led_scan_rows=scan, led_scan_cols=scan, tile_overlap=8) if n == 64 else
           fpm.OpticalConfig(tile_size=n, tile_overlap=0, upsample=4, led_scan_rows=scan, led_scan_cols=scan))
    fs, _, seq, _ = dataset(cfg, fov=fov, seed=77, defocus_um=4.0)
    specs = fpm.partition_tiles(fs.width(), fs.height(), cfg)
    dz = list(np.linspace(-6, 6, len(specs)))
    opt = fpm.RunOptions(iters=iters, mode=mode, tile_defocus_um=dz)
    monkeypatch.delenv("FPM_B200_JITTER", raising=False)
    ref = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
    res_ref = np.array([m.pass_mean_residual for m in ref.tile_metrics])
    for seed in (1, 2, 3):
        monkeypatch.setenv("FPM_B200_JITTER", f"3000:{seed}")
        got = fpm.run_offline(fs, cfg, seq, opt, engine=fpm.Engine(0), stitch=False)
        assert np.array_equal(got.tiles, ref.tiles), (case, seed)
        assert np.array_equal(np.array([m.pass_mean_residual for m in got.tile_metrics]), res_ref), (case, seed)
        if mode == "epry":
            assert np.array_equal(got.pupils, ref.pupils), (case, seed)
