"""The C++ drop-in (include/fpm_b200.hpp) re-runs the reference's own tests
through the reference's API names; on the GPU its outputs are compared with
the oracle."""
import os
import struct
import subprocess

import numpy as np
import pytest

from tests.helpers import amp_phase_rel, dataset, gpu_cfg, orc_cfg

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "api_check")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)


def test_cpp_api_geometry_cpu():
    _build()
    out = subprocess.run([BIN, "cpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "OK" in out.stdout


def _read_field(path):
    with open(path, "rb") as f:
        r, c = struct.unpack("ii", f.read(8))
        return np.frombuffer(f.read(), np.float64).view(np.complex128).reshape(r, c)


@pytest.mark.gpu
@pytest.mark.parametrize("scan,order,iters", [(3, "spiral", 3), (7, "raster", 2)])
def test_cpp_api_reconstruction_gpu(orc, tmp_path, scan, order, iters):
    _build()
    cfg = gpu_cfg(led_scan_rows=scan, led_scan_cols=scan, tile_overlap=8)
    fs, ofs, seq, _ = dataset(cfg, order=order, fov=120, seed=40 + scan)
    d = str(tmp_path)
    with open(os.path.join(d, "cfg.txt"), "w") as f:
        f.write(f"64 8 4 {scan} {scan} {iters} {1 if order == 'raster' else 0}\n")
    with open(os.path.join(d, "frames.bin"), "wb") as f:
        F, H, W = fs.images.shape
        f.write(struct.pack("iii", F, H, W))
        f.write(np.asarray(fs.leds, np.int32).tobytes())
        f.write(np.ascontiguousarray(fs.images, np.uint16).tobytes())
    out = subprocess.run([BIN, "gpu", d], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    hr = _read_field(os.path.join(d, "hr.bin"))
    ref = orc.reconstruct_tile(ofs, orc_cfg(cfg), iters, seq)
    amp, ph = amp_phase_rel(hr, ref.hr)
    assert amp < 1e-4 and ph < 1e-4, (amp, ph)
    resid = np.fromfile(os.path.join(d, "resid.bin"), np.float64)
    assert np.allclose(resid, ref.residuals, rtol=1e-3)
    st = _read_field(os.path.join(d, "stitched.bin"))
    ref_st = orc.run_offline(ofs, orc_cfg(cfg), seq, iters).stitched
    amp, ph = amp_phase_rel(st, ref_st)
    assert amp < 1e-4 and ph < 1e-4, (amp, ph)
