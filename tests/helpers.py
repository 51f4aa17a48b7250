"""Shared fixtures: physical parity stacks from the oracle's forward model and
the parity metrics of the north star (relative L2 of amplitude and phase)."""
from __future__ import annotations

import numpy as np

import paper_2203_02507_b200 as fpm
from oracle import oracle as orc


def gpu_cfg(**kw) -> fpm.OpticalConfig:
    base = dict(tile_size=64, tile_overlap=8, upsample=4, led_scan_rows=3, led_scan_cols=3)
    base.update(kw)
    return fpm.OpticalConfig(**base)


def orc_cfg(cfg: fpm.OpticalConfig) -> orc.Optics:
    return orc.Optics(**{f: getattr(cfg, f) for f in orc.Optics.__dataclass_fields__})


def dataset(cfg: fpm.OpticalConfig, order: str = "spiral", fov: int | None = None, seed: int = 1,
            defocus_um: float = 0.0, kind: str = "composite", noise=None):
    """simulate_dataset(synth_object(kind, FOV*up, seed)) in the oracle -> (FrameSet, seq, object)."""
    oc = orc_cfg(cfg)
    fov = fov or cfg.tile_size
    size = max(fov * cfg.upsample, 256)
    obj = orc.synth_object(kind, size, seed)[: fov * cfg.upsample, : fov * cfg.upsample]
    seq = orc.led_sequence(order, oc)
    fs = orc.simulate_dataset(obj, seq, oc, noise=noise, defocus_um=defocus_um)
    return fpm.FrameSet(fs.images, list(fs.leds), fs.timestamps), orc.FrameStack(fs.images, list(fs.leds)), seq, obj


def rel_l2(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def amp_phase_rel(a, b):
    """(amplitude rel-L2, amplitude-weighted phase rel-L2) of field a against b."""
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    amp = np.linalg.norm(np.abs(a) - np.abs(b)) / np.linalg.norm(np.abs(b))
    dphi = np.angle(a * np.conj(b))
    ph = np.sqrt(np.sum(np.abs(b) ** 2 * dphi ** 2) / np.sum(np.abs(b) ** 2))
    return float(amp), float(ph)
