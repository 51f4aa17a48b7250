"""The `fpm` command line (paper_2203_02507_b200/cli.py) against the reference's
fpm_main.cpp contract: subcommands and options, exit codes 2 (config / command
line), 3 (data / IO), 4 (unsafe lag) (fpm_main.cpp:21-23, :341-353), the
timings CSV columns (parallel.cpp:113-122) and the output files of
`reconstruct` (tile_<y0>_<x0>.cfi, stitched.cfi, timings.csv, report.json).
CPU cases exercise parsing and the host-side error paths; the GPU cases run
reconstruct / bench / stitch / export end to end."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2203_02507_b200 as fpm
from paper_2203_02507_b200 import cli
from tests.helpers import dataset, gpu_cfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*argv):
    return subprocess.run([sys.executable, "-m", "paper_2203_02507_b200", *argv], capture_output=True, text=True,
                          cwd=ROOT, timeout=600)


def test_bad_command_line_exits_2():
    r = _run("reconstruct", "--data", "x")  # --out missing
    assert r.returncode == cli.EXIT_CONFIG, r.stderr
    assert _run("frobnicate").returncode == cli.EXIT_CONFIG
    assert _run().returncode == cli.EXIT_CONFIG


def test_missing_dataset_exits_3(tmp_path):
    r = _run("reconstruct", "--data", str(tmp_path / "nope"), "--out", str(tmp_path / "o"))
    assert r.returncode == cli.EXIT_DATA
    assert "missing manifest.json" in r.stderr


def test_bench_tile_count_beyond_partition_exits_2(tmp_path):
    cfg = gpu_cfg(led_scan_rows=3, led_scan_cols=3)
    fs, _, _, _ = dataset(cfg, fov=120, seed=3)
    fpm.write_dataset(tmp_path / "d", fs, cfg)
    r = _run("bench", "--data", str(tmp_path / "d"), "--tiles", "1,99", "--out", str(tmp_path / "t.csv"))
    assert r.returncode == cli.EXIT_CONFIG
    assert "exceeds partition of 4" in r.stderr
    assert _run("bench", "--data", str(tmp_path / "d"), "--tiles", "a,b", "--out",
                str(tmp_path / "t.csv")).returncode == cli.EXIT_CONFIG


def test_stitch_tile_list_errors_exit_3(tmp_path):
    lst = tmp_path / "tiles.list"
    lst.write_text("")
    r = _run("stitch", "--inputs", str(lst), "--out", str(tmp_path / "o.cfi"))
    assert r.returncode == cli.EXIT_DATA and "tile list is empty" in r.stderr
    lst.write_text("0 zero a.cfi\n")
    r = _run("stitch", "--inputs", str(lst), "--out", str(tmp_path / "o.cfi"))
    assert r.returncode == cli.EXIT_DATA and "malformed tile list line" in r.stderr
    assert _run("stitch", "--inputs", str(tmp_path / "none"), "--out", "x").returncode == cli.EXIT_DATA


def test_nonempty_output_directory_refused(tmp_path):
    cfg = gpu_cfg(led_scan_rows=3, led_scan_cols=3)
    fs, _, _, _ = dataset(cfg, fov=64, seed=3)
    fpm.write_dataset(tmp_path / "d", fs, cfg)
    (tmp_path / "o").mkdir()
    (tmp_path / "o" / "keep").write_text("x")
    r = _run("reconstruct", "--data", str(tmp_path / "d"), "--out", str(tmp_path / "o"))
    assert r.returncode == cli.EXIT_DATA and "use --force" in r.stderr


def test_timing_csv_format():
    t = fpm.engine.TimingRow("bench", "offline", 2, 1, 4, 1, 0.1234567, 0.0308642)
    assert cli.CSV_HEADER == "run_id,mode,workers,lag,tiles,iters,wall_s,per_tile_mean_s"
    assert cli.timing_csv_row(t) == "bench,offline,2,1,4,1,0.123457,0.0308642"


@pytest.mark.gpu
def test_reconstruct_outputs_and_metrics(tmp_path):
    cfg = gpu_cfg(led_scan_rows=5, led_scan_cols=5, tile_overlap=8)
    fs, _, _, obj = dataset(cfg, fov=120, seed=7)
    fpm.write_dataset(tmp_path / "d", fs, cfg, object_truth=obj)
    r = _run("reconstruct", "--data", str(tmp_path / "d"), "--out", str(tmp_path / "o"), "--iters", "2")
    assert r.returncode == 0, r.stderr
    names = sorted(os.listdir(tmp_path / "o"))
    assert names == ["report.json", "stitched.cfi", "tile_000_000.cfi", "tile_000_056.cfi", "tile_056_000.cfi",
                     "tile_056_056.cfi", "timings.csv"]
    lines = (tmp_path / "o" / "timings.csv").read_text().splitlines()
    assert lines[0] == cli.CSV_HEADER and lines[1].startswith("reconstruct,offline,1,1,4,2,")
    rep = json.loads((tmp_path / "o" / "report.json").read_text())
    assert rep["command"] == "reconstruct" and len(rep["metrics"]["pass_mean_residual"]) == 4
    assert rep["metrics"]["amplitude_rmse_vs_truth"] < 0.2
    # the CLI's files equal the API's results bit for bit
    res = fpm.run_offline(fpm.read_dataset(tmp_path / "d").frames, cfg, fpm.led_sequence("spiral", cfg),
                          fpm.RunOptions(iters=2))
    assert np.array_equal(fpm.read_cfi(tmp_path / "o" / "stitched.cfi"), res.stitched.astype(np.complex128))
    # unsafe lag -> 4 (UnsafeLagError, fpm_main.cpp:344-346)
    r = _run("reconstruct", "--data", str(tmp_path / "d"), "--out", str(tmp_path / "o2"), "--force-pipeline",
             "--lag", "1")
    assert r.returncode == cli.EXIT_UNSAFE, r.stderr
    # stitch + export of the CLI's own tiles
    lst = tmp_path / "tiles.list"
    lst.write_text("".join(f"{x} {y} {tmp_path / 'o' / f'tile_{y:03d}_{x:03d}.cfi'}\n"
                           for y in (0, 56) for x in (0, 56)))
    cj = tmp_path / "cfg.json"
    fpm.write_config(cj, fpm.AppConfig(optics=cfg))
    r = _run("stitch", "--inputs", str(lst), "--out", str(tmp_path / "s.cfi"), "--config", str(cj))
    assert r.returncode == 0, r.stderr
    assert np.array_equal(fpm.read_cfi(tmp_path / "s.cfi"), fpm.read_cfi(tmp_path / "o" / "stitched.cfi"))
    r = _run("export", "--in", str(tmp_path / "s.cfi"), "--amplitude", str(tmp_path / "a.pgm"))
    assert r.returncode == 0 and (tmp_path / "a.pgm").exists()


@pytest.mark.gpu
def test_bench_sweep(tmp_path):
    cfg = gpu_cfg(led_scan_rows=3, led_scan_cols=3, tile_overlap=8)
    fs, _, _, _ = dataset(cfg, fov=120, seed=8)
    fpm.write_dataset(tmp_path / "d", fs, cfg)
    r = _run("bench", "--data", str(tmp_path / "d"), "--workers", "1,2", "--tiles", "1,4", "--out",
             str(tmp_path / "t.csv"))
    assert r.returncode == 0, r.stderr
    rows = (tmp_path / "t.csv").read_text().splitlines()
    assert rows[0] == cli.CSV_HEADER and len(rows) == 5
    assert [r_.split(",")[2:5] for r_ in rows[1:]] == [["1", "1", "1"], ["1", "1", "4"], ["2", "1", "1"],
                                                       ["2", "1", "4"]]
    assert "tiles=4 speedup: x1" in r.stdout
