"""bench.py's strong-scaled multi-rank step (BASELINE config 4) end to end:
torchrun with 2 ranks on the one available GPU, host-side (gloo) collectives,
every rank writing its band of rank 0's mosaic through CUDA IPC. A functional
check of the JSON contract of the N > 1 line — the numbers are not a
measurement (both ranks share one GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_strong_scaled_bench_line_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--dist-backend", "gloo"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["steps"] == 2
    assert d["config"]["baseline_config"] == 4 and d["config"]["ranks"] == 2
    assert d["config"]["updates_per_step_all_ranks"] == 2304000
    assert abs(d["value"] - 2304000 / d["full_recon_s"]) / d["value"] < 1e-9
    assert "NVLink" in d["parallelism"] and "mosaic" in d["step"]
    assert d["residuals_finite"] is True
    e2e = d["e2e"]
    assert e2e["h2d_bytes_per_step"] == 225 * 2048 * 2048 * 2 and e2e["d2h_bytes_per_step"] > 8192 * 8192 * 8
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
    assert d["roofline"]["measured_on"] == "rank 0's band"
