"""GPU forward model: simulate_dataset (forward.cpp:172-282) on the device.

SURVEY §8(f) rank 1: the fixture generator for physical parity stacks at
BASELINE scale (config 3: 1,024 tiles x 225 LEDs; config 5: a 4 GiB HR object),
which the CPU restatement needs tens of core-minutes for. It follows the
reference step for step, in float64/complex128 so the quantised u16 frames
match the double-precision oracle:

* per tile, an HR crop with even guard bands of up to n/2 LR pixels per side
  (forward.cpp:214-224), its centred spectrum (field.cpp:48-56);
* per LED, the (ph x pw) sub-aperture at the LED's offset on the crop's own
  frequency grid (dky = 1/(ph dx), forward.cpp:226-233) times the coherent
  transfer function — the NA disk, with the defocus phase
  exp(i 2 pi z sqrt(1/lambda^2 - |f|^2)) (forward.cpp:234-245) — then |ifft2|^2;
* the feathered assembly: linear ramps across each overlap, normalised by the
  summed weights (forward.cpp:187-205, :256);
* the grey scale anchored to the on-axis frame (else the brightest,
  forward.cpp:259-268) and quantisation with lround + clamp (forward.cpp:145-160).

All LEDs of a tile run as one batched transform. On the device the 2-D
transforms are this repo's complex128 Stockham kernel (`fft_c128.cu`, radix
2/3/4/5: the guard-banded grids are 96 / 120 / 384 / 480 / 512 ... points, not
the power-of-two sides of the reconstruction kernels); shifts, the transfer
function, |.|^2 and the feathered assembly are elementwise torch ops. This is
the fixture path, not the reconstruction hot path. Photon noise,
when requested, draws from torch's Poisson generator, not the reference's
std::mt19937_64 stream, so noisy frames are statistically — not bitwise —
equivalent.
"""
from __future__ import annotations

import numpy as np

from .engine import (DataError, FrameSet, OpticalConfig, partition_arrays, scan_leds,  # noqa: F401
                     tile_origins)


def _lround(x):
    """C lround (half away from zero) for numpy or torch arrays."""
    import torch
    if isinstance(x, torch.Tensor):
        a = torch.abs(x)
        r = torch.where(a - torch.floor(a) == 0.5, torch.ceil(a), torch.round(a))
        return torch.sign(x) * r
    a = np.abs(x)
    r = np.where(a - np.floor(a) == 0.5, np.ceil(a), np.round(a))
    return np.sign(x) * r


def _axis_weights(origins, n):
    """Feathering ramps of one axis (forward.cpp:187-205)."""
    w = np.ones((len(origins), n))
    for k, o in enumerate(origins):
        if k > 0:
            prev_end = origins[k - 1] + n
            for x in range(o, min(prev_end, o + n)):
                w[k, x - o] *= (x - o + 1) / (prev_end - o + 1)
        if k + 1 < len(origins):
            nxt = origins[k + 1]
            for x in range(max(nxt, o), o + n):
                w[k, x - o] *= (o + n - x) / (o + n - nxt + 1)
    return w


def fft2_c128(x, inverse=False):
    """2-D FFT over the last two axes of a complex128 CUDA tensor on this repo's
    kernel (fpmgpu_fft2_c128: Stockham radix 2/3/4/5 in double, any side with
    factors 2, 3, 5 up to 4096); numpy / torch.fft conventions (the inverse
    divides by rows * cols)."""
    import ctypes as C

    import torch
    from ._lib import check, lib
    from .engine import default_engine
    y = x.contiguous().clone()
    rows, cols = int(y.shape[-2]), int(y.shape[-1])
    batch = int(y.numel() // max(rows * cols, 1))
    eng = default_engine(y.device.index if y.device.index is not None else torch.cuda.current_device())
    check(lib().fpmgpu_fft2_c128(eng.handle, C.c_void_p(y.data_ptr()), batch, rows, cols, 1 if inverse else 0,
                                 C.c_void_p(torch.cuda.current_stream(y.device).cuda_stream)))
    return y


def _centered(x, inverse=False):
    """fftshift(FFT(ifftshift(x))) over the last two axes (field.cpp:48-87); the
    inverse divides by rows * cols. On the device the transform is this repo's
    FP64 kernel (fft2_c128); the CPU path (device="cpu", the CPU tests) uses
    torch.fft."""
    import torch
    y = torch.fft.ifftshift(x, dim=(-2, -1))
    if y.is_cuda:
        y = fft2_c128(y, inverse)
    else:
        y = torch.fft.ifft2(y) if inverse else torch.fft.fft2(y)
    return torch.fft.fftshift(y, dim=(-2, -1))


def simulate_dataset(obj, seq, cfg: OpticalConfig, noise: tuple | None = None, defocus_um: float = 0.0,
                     device: str = "cuda") -> FrameSet:
    """simulate_dataset(object_hr, seq, cfg, noise, defocus_um) -> FrameSet (forward.cpp:172-282).

    obj: complex HR object [FOV_h*up, FOV_w*up] (numpy or torch); seq: LED
    (row, col) sequence; noise: None or (photons, seed)."""
    import torch
    cfg.validate()
    up, n = cfg.upsample, cfg.tile_size
    o = torch.as_tensor(obj).to(device=device, dtype=torch.complex128)
    if o.shape[0] % up or o.shape[1] % up:
        raise DataError("object dimensions must be a multiple of upsample")
    fov_h, fov_w = o.shape[0] // up, o.shape[1] // up
    leds = scan_leds(cfg)
    index = {led: k for k, led in enumerate(leds)}
    seq = [tuple(s) for s in seq]
    for s in seq:
        if s not in index:
            raise DataError(f"sequence LED {s} is outside the scan")
    sel = np.array([index[s] for s in seq], np.int64)
    xy, _, kv, _ = partition_arrays(fov_w, fov_h, cfg, leds)
    xs, ys = tile_origins(fov_w, n, cfg.tile_overlap), tile_origins(fov_h, n, cfg.tile_overlap)
    wx, wy = _axis_weights(xs, n), _axis_weights(ys, n)
    L = len(seq)
    buffers = torch.zeros((L, fov_h, fov_w), dtype=torch.float64, device=device)
    wsum = torch.zeros((fov_h, fov_w), dtype=torch.float64, device=device)
    dx = cfg.camera_pixel / cfg.magnification
    cutoff = cfg.objective_na / cfg.wavelength
    inv_l2 = 1.0 / (cfg.wavelength * cfg.wavelength)
    for ti in range(len(xy)):
        x0, y0 = int(xy[ti, 0]), int(xy[ti, 1])
        ci, ri = ti % len(xs), ti // len(xs)
        ml, mr = min(n // 2, x0) & ~1, min(n // 2, fov_w - x0 - n) & ~1
        mt, mb = min(n // 2, y0) & ~1, min(n // 2, fov_h - y0 - n) & ~1
        pw, ph = n + ml + mr, n + mt + mb
        PW, PH = pw * up, ph * up
        crop = o[(y0 - mt) * up:(y0 - mt) * up + PH, (x0 - ml) * up:(x0 - ml) * up + PW]
        spectrum = _centered(crop)
        dky, dkx = 1.0 / (ph * dx), 1.0 / (pw * dx)
        w2 = torch.as_tensor(np.outer(wy[ri], wx[ci]), device=device)
        wsum[y0:y0 + n, x0:x0 + n] += w2
        oy = _lround(kv[ti, sel, 1] / dky).astype(np.int64)
        ox = _lround(kv[ti, sel, 0] / dkx).astype(np.int64)
        r0, c0 = PH // 2 + oy - ph // 2, PW // 2 + ox - pw // 2
        if (r0 < 0).any() or (c0 < 0).any() or (r0 + ph > PH).any() or (c0 + pw > PW).any():
            raise DataError("illumination NA too high for upsample factor")
        fy = (torch.arange(ph, device=device, dtype=torch.float64) - ph // 2) * dky
        fx = (torch.arange(pw, device=device, dtype=torch.float64) - pw // 2) * dkx
        fr = torch.hypot(fy[:, None], fx[None, :])
        ctf = (fr <= cutoff).to(torch.complex128)
        if defocus_um != 0.0:
            kz = torch.sqrt(torch.clamp(inv_l2 - fr * fr, min=0.0))
            ctf = ctf * torch.polar(torch.ones_like(kz), 2.0 * np.pi * defocus_um * kz)
        rows = torch.as_tensor(r0, device=device)[:, None] + torch.arange(ph, device=device)[None, :]
        cols = torch.as_tensor(c0, device=device)[:, None] + torch.arange(pw, device=device)[None, :]
        blocks = spectrum[rows[:, :, None], cols[:, None, :]] * ctf
        patch = _centered(blocks, inverse=True).abs().square()
        buffers[:, y0:y0 + n, x0:x0 + n] += w2 * patch[:, mt:mt + n, ml:ml + n]
    buffers /= wsum
    center = (cfg.center_row, cfg.center_col)
    peak = 0.0
    for li in range(L):  # anchor to the on-axis frame when present (forward.cpp:259-268)
        if seq[li] == center:
            peak = float(buffers[li].max())
            break
        peak = max(peak, float(buffers[li].max()))
    if peak <= 0:
        raise DataError("dataset is identically zero")
    counts = buffers * (0.8 * 65535.0 / peak)
    if noise is not None:
        photons, seed = noise
        g = torch.Generator(device=device)
        g.manual_seed(int(seed))
        mean = torch.clamp(counts / 65535.0 * photons, min=0.0)
        counts = torch.poisson(mean, generator=g) / photons * 65535.0
    images = torch.clamp(_lround(counts), 0, 65535).to(torch.int32).cpu().numpy().astype(np.uint16)
    step = cfg.acq_pattern_delay + cfg.acq_exposure
    return FrameSet(images, list(seq), np.array([(li + 1) * step for li in range(L)]))
