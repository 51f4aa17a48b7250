"""Generate the golden fixtures under tests/golden/ from the CPU oracle.

The reference (/root/reference/proj) cannot be built in this image (no Eigen),
so its outputs cannot be recorded directly; these fixtures freeze the oracle's
outputs on physically simulated stacks (its own forward model,
forward.cpp:172-282) and the reference's known-answer literals. The oracle is
itself pinned by tests/test_oracle_pins.py against the reference's tests.

  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402

CASES = {
    # name: (tile, overlap, scan, fov, seed, defocus_sim, order, iters, mode, hr_stride)
    "toy3x3_gs": (64, 8, 3, 64, 4, 0.0, "spiral", 3, "gs", 1),
    "c1_7x7_gs": (64, 0, 7, 64, 1, 0.0, "spiral", 5, "gs", 1),
    "epry_9x9_defocus25": (64, 0, 9, 64, 5, 25.0, "spiral", 3, "epry", 1),
    "n128_7x7_epry": (128, 0, 7, 128, 2, 15.0, "spiral", 2, "epry", 4),
}

MOSAIC = ("mosaic120_5x5_gs", 64, 8, 5, 120, 32, 2)


def case(name):
    tile, ov, scan, fov, seed, dz, order, iters, mode, stride = CASES[name]
    cfg = orc.Optics(tile_size=tile, tile_overlap=ov, upsample=4, led_scan_rows=scan, led_scan_cols=scan)
    size = max(fov * 4, 256)
    obj = orc.synth_object("composite", size, seed)[: fov * 4, : fov * 4]
    seq = orc.led_sequence(order, cfg)
    fs = orc.simulate_dataset(obj, seq, cfg, defocus_um=dz)
    r = orc.reconstruct_tile(fs, cfg, iters, seq, mode=mode)
    return cfg, fs, seq, r, stride


def literals():
    c = orc.Optics()
    toy = orc.toy_cfg()
    fx, fy = orc.illumination_wavevector((32, 33), (0, 0), c)
    return {
        "one_pitch_fx": {"value": fx, "ref": "proj/tests/test_optics.cpp:38-46", "expect": -0.0573463, "rel": 1e-5},
        "one_pitch_offset_px": {"value": list(orc.spectrum_offset_px((fx, fy), c)), "expect": [0, -18],
                                "ref": "proj/tests/test_forward.cpp:92-98"},
        "pupil_radius_256": {"value": orc.build_pupil(c, 256)[1], "expect": 58.514, "rel": 1e-4,
                             "ref": "proj/tests/test_optics.cpp:79-101"},
        "synthesized_na": {"value": orc.synthesized_na(c), "expect": 0.34762, "rel": 1e-4,
                           "ref": "proj/tests/test_optics.cpp:119-124"},
        "tile_origins_2048_256_26": {"value": orc.tile_origins(2048, 256, 26),
                                     "expect": [0, 230, 460, 690, 920, 1150, 1380, 1610, 1792],
                                     "ref": "proj/tests/test_parallel.cpp:143-149"},
        "toy_min_safe_lag": {"value": orc.min_safe_lag_tile(toy, 64, 64, 0, orc.led_sequence("spiral", toy)),
                             "expect": 9, "ref": "proj/tests/test_parallel.cpp:56-62"},
        "spiral_3x3": {"value": [list(x) for x in orc.sequence_offsets("spiral", 3, 3)],
                       "expect": [[0, 0], [0, 1], [-1, 1], [-1, 0], [-1, -1], [0, -1], [1, -1], [1, 0], [1, 1]],
                       "ref": "proj/tests/test_recon.cpp:22-27"},
    }


def main():
    for name in CASES:
        cfg, fs, seq, r, stride = case(name)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), frames=fs.images, leds=np.asarray(fs.leds, np.int32),
                            seq=np.asarray(seq, np.int32), hr=r.hr[::stride, ::stride].astype(np.complex64),
                            hr_stride=stride, residuals=r.residuals, pupil=r.pupil.astype(np.complex64))
        print(name, fs.images.shape, r.residuals)
    name, tile, ov, scan, fov, seed, iters = MOSAIC
    cfg = orc.Optics(tile_size=tile, tile_overlap=ov, upsample=4, led_scan_rows=scan, led_scan_cols=scan)
    obj = orc.synth_object("composite", fov * 4, seed)
    seq = orc.led_sequence("spiral", cfg)
    fs = orc.simulate_dataset(obj, seq, cfg)
    res = orc.run_offline(fs, cfg, seq, iters)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), frames=fs.images, leds=np.asarray(fs.leds, np.int32),
                        seq=np.asarray(seq, np.int32), stitched=res.stitched[::2, ::2].astype(np.complex64),
                        residuals=res.residuals)
    print(name, res.stitched.shape)
    with open(os.path.join(HERE, "reference_literals.json"), "w") as f:
        json.dump(literals(), f, indent=1)


if __name__ == "__main__":
    main()
