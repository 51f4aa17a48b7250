"""bench.py's JSON-line contract, on the one arm that runs without a GPU: the
reference arm (`--impl reference`, the oracle's threaded run_offline on a
bounded sample of BASELINE config 3)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "LED-updates/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["config"]["baseline_config"] == 3
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and "sample" in cb
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the reference arm runs the oracle restatement only: the product library is never mapped
    assert d["repo_native_libs_loaded"] == ["oracle/lib/libfpm_oracle.so"], d["repo_native_libs_loaded"]
    assert d["scaling"] == "strong" and d["config"]["updates_per_step_all_ranks"] == 2304000


def test_config_blocks_identical_across_arms():
    """Both arms print the same config block for the same (N, scaling): the
    driver's ratio needs same_config."""
    sys.path.insert(0, ROOT)
    import bench
    W = bench.WORKLOADS[3]
    for world in (1, 2, 8):
        for scaling in ("strong", "weak"):
            a = bench.config_block(W, world, scaling)
            assert a == bench.config_block(W, world, scaling)
            assert a["updates_per_step_all_ranks"] == W.updates * (world if scaling == "weak" else 1)
    assert bench.config_block(W, 8, "strong")["baseline_config"] == 4
