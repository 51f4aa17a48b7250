"""`fpm` command line on the B200 engine: the reference's
`reconstruct`, `bench`, `stitch` and `export` subcommands
(/root/reference/proj/tools/fpm_main.cpp:117-186, :188-222, :224-234, :236-281)
with the same options, outputs and exit codes — 2 for configuration errors
(and bad command lines), 3 for data / IO errors, 4 for an unsafe pipeline lag
(fpm_main.cpp:21-23, :341-353).

    python -m paper_2203_02507_b200 reconstruct --data DIR --out DIR [--iters N] ...
    python -m paper_2203_02507_b200 bench --data DIR --out timings.csv [--workers 1,2] [--tiles 1,4]

Outputs match the reference's byte layouts: one CFI per tile named
tile_<y0>_<x0>.cfi, stitched.cfi, timings.csv with the reference's columns
(parallel.cpp:113-122) and report.json. `simulate` (a fixture generator off the
reconstruction path) is not part of this CLI.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import engine as E
from . import formats as F
from ._lib import ConfigError, DataError, UnsafeLagError

EXIT_CONFIG, EXIT_DATA, EXIT_UNSAFE = 2, 3, 4
CSV_HEADER = "run_id,mode,workers,lag,tiles,iters,wall_s,per_tile_mean_s"


def default_workers() -> int:
    """fpm_main.cpp:25-31: FPM_WORKERS, else 1."""
    try:
        w = int(os.environ.get("FPM_WORKERS", ""))
        return w if w >= 1 else 1
    except ValueError:
        return 1


def parse_int_list(s: str) -> list:
    try:
        out = [int(x) for x in s.split(",") if x != ""]
    except ValueError:
        raise ConfigError(f"not an integer list: {s}") from None
    if not out:
        raise ConfigError("empty list: " + s)
    return out


def _fmt(v) -> str:
    """std::ostream's default float format (6 significant digits, %g)."""
    return f"{v:g}" if isinstance(v, float) else str(v)


def timing_csv_row(t: E.TimingRow) -> str:
    return ",".join(_fmt(x) for x in (t.run_id, t.mode, t.workers, t.lag, t.tiles, t.iters, float(t.wall_s),
                                      float(t.per_tile_mean_s)))


def _timing_json(t: E.TimingRow) -> dict:
    return {"run_id": t.run_id, "mode": t.mode, "workers": t.workers, "lag": t.lag, "tiles": t.tiles,
            "iters": t.iters, "wall_s": t.wall_s, "per_tile_mean_s": t.per_tile_mean_s}


def write_report(out_dir, command, cfg: F.AppConfig, rows, metrics, outputs) -> None:
    """fpm_main.cpp:42-64."""
    rep = {"command": command, "config": json.loads(F.config_to_json(cfg)),
           "timing": [_timing_json(r) for r in rows], "metrics": metrics, "outputs": outputs}
    with open(os.path.join(out_dir, "report.json"), "w") as f:
        f.write(json.dumps(rep, indent=2) + "\n")


def _prepare_out(out: str, force: bool) -> None:
    if os.path.exists(out) and os.listdir(out) and not force:
        raise DataError(f"output directory not empty (use --force): {out}")
    os.makedirs(out, exist_ok=True)


# ------------------------------------------------------------------ truth metrics (metrics.cpp:7-57)
def _fft2c(x):
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x)))


def _ifft2c(x):
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(x)))


def band_limit(field_, na: float, cfg: E.OpticalConfig) -> np.ndarray:
    n = field_.shape[0]
    if field_.shape[1] != n:
        raise DataError("band_limit expects a square field")
    dk = 1.0 / (cfg.tile_size * cfg.dx_obj())
    radius = (na / cfg.wavelength) / dk
    spec = _fft2c(np.asarray(field_, np.complex128))
    i, j = np.mgrid[0:n, 0:n]
    spec[np.hypot(i - n // 2, j - n // 2) > radius] = 0
    return _ifft2c(spec)


def global_alignment(recon, truth) -> complex:
    r = np.asarray(recon, np.complex128)
    den = float(np.sum(np.abs(r) ** 2))
    if den <= 0:
        raise DataError("global_alignment: zero reconstruction")
    return complex(np.sum(np.asarray(truth, np.complex128) * np.conj(r)) / den)


def amplitude_rmse(a, b) -> float:
    return float(np.sqrt(np.mean((np.abs(a) - np.abs(b)) ** 2)))


def phase_rmse(a, b) -> float:
    d = np.angle(a) - np.angle(b)
    d = (d + np.pi) % (2 * np.pi) - np.pi
    return float(np.sqrt(np.mean(d ** 2)))


# ------------------------------------------------------------------ subcommands
def cmd_reconstruct(a) -> int:
    """fpm_main.cpp:117-186."""
    ds = F.read_dataset(a.data)
    cfg = F.AppConfig(optics=ds.cfg)
    cfg_path = os.path.join(a.data, "config.json")
    if os.path.exists(cfg_path):
        cfg.run = F.read_config(cfg_path).run
    if a.iters > 0:
        cfg.run.iters = a.iters
    if a.order:
        cfg.run.order = a.order
    if a.workers > 0:
        cfg.run.workers = a.workers
    elif cfg.run.workers == 1:
        cfg.run.workers = default_workers()
    if a.mode:
        cfg.run.mode = a.mode
    if a.online_delay >= 0:
        cfg.run.online_delay = a.online_delay
    if a.lag != "auto":
        try:
            cfg.run.lag = int(a.lag)
        except ValueError:
            raise ConfigError(f"--lag must be auto or an integer: {a.lag}") from None
    _prepare_out(a.out, a.force)
    opt = E.RunOptions(iters=cfg.run.iters, workers=cfg.run.workers, lag=cfg.run.lag,
                       force_unsafe_lag=a.unsafe_lag, force_pipeline=a.force_pipeline,
                       defocus_um=cfg.run.defocus_um, max_tiles=a.tiles if a.tiles > 0 else None)
    if cfg.run.mode == "online" and cfg.run.defocus_candidates_um:
        raise ConfigError("online mode requires explicit per-tile defocus, not a search")
    if cfg.run.mode not in ("offline", "online"):
        raise ConfigError(f"unknown run mode: {cfg.run.mode}")
    seq = E.led_sequence(cfg.run.order, cfg.optics)
    if cfg.run.mode == "online":
        res = E.run_online(ds.frames, cfg.optics, seq, opt, cfg.run.online_delay)
    else:
        res = E.run_offline(ds.frames, cfg.optics, seq, opt)
    res.timing.run_id = "reconstruct"
    outputs = []
    for spec, tile in zip(res.specs, res.tiles):
        name = f"tile_{spec.y0:03d}_{spec.x0:03d}.cfi"
        F.write_cfi(os.path.join(a.out, name), tile)
        outputs.append(name)
    metrics = {}
    if res.stitched is not None and res.stitched.size > 0:
        F.write_cfi(os.path.join(a.out, "stitched.cfi"), res.stitched)
        outputs.append("stitched.cfi")
    metrics["pass_mean_residual"] = [m.pass_mean_residual for m in res.tile_metrics]
    if ds.object_truth and res.stitched is not None and res.stitched.size > 0:
        truth = F.read_cfi(ds.object_truth)
        if truth.shape == res.stitched.shape and truth.shape[0] == truth.shape[1]:
            limited = band_limit(truth, E.synthesized_na(cfg.optics), cfg.optics)
            st = res.stitched.astype(np.complex128)
            aligned = st * global_alignment(st, limited)
            metrics["amplitude_rmse_vs_truth"] = amplitude_rmse(aligned, limited)
            metrics["phase_rmse_vs_truth"] = phase_rmse(aligned, limited)
    if cfg.run.mode == "online":
        metrics["acquisition_s"] = res.acquisition_s
    with open(os.path.join(a.out, "timings.csv"), "w") as f:
        f.write(CSV_HEADER + "\n" + timing_csv_row(res.timing) + "\n")
    write_report(a.out, "reconstruct", cfg, [res.timing], metrics, outputs)
    print(f"reconstructed {len(res.tiles)} tile(s) in {_fmt(float(res.timing.wall_s))} s")
    return 0


def cmd_stitch(a) -> int:
    """fpm_main.cpp:188-222: tile list lines '<x0_lr> <y0_lr> <path.cfi>'."""
    cfg = F.read_config(a.config) if a.config else F.AppConfig()
    try:
        with open(a.inputs) as f:
            lines = f.read().splitlines()
    except OSError:
        raise DataError(f"cannot open tile list {a.inputs}") from None
    tiles, specs = [], []
    for line in lines:
        if not line:
            continue
        parts = line.split()
        if len(parts) < 3:
            raise DataError("malformed tile list line: " + line)
        try:
            x0, y0 = int(parts[0]), int(parts[1])
        except ValueError:
            raise DataError("malformed tile list line: " + line) from None
        specs.append(E.TileSpec(x0, y0, cfg.optics.tile_size))
        tiles.append(F.read_cfi(parts[2]))
    if not tiles:
        raise DataError("tile list is empty")
    out = tiles[0] if len(tiles) == 1 else E.stitch_mosaic(np.stack(tiles), specs, cfg.optics)
    F.write_cfi(a.out, out)
    print(f"stitched {len(tiles)} tile(s) -> {out.shape[1]}x{out.shape[0]}")
    return 0


def cmd_export(a) -> int:
    """fpm_main.cpp:224-234."""
    f = F.read_cfi(a.input)
    if a.amplitude:
        F.export_view(f, "amplitude", a.amplitude)
    if a.phase:
        F.export_view(f, "phase", a.phase)
    return 0


def cmd_bench(a) -> int:
    """fpm_main.cpp:236-281: run_offline over workers x tile counts, timings CSV."""
    ds = F.read_dataset(a.data)
    cfg = ds.cfg
    seq = E.led_sequence("spiral", cfg)
    workers = parse_int_list(a.workers)
    tile_counts = parse_int_list(a.tiles)
    partition = E.partition_tiles(ds.frames.width(), ds.frames.height(), cfg)
    for t in tile_counts:
        if t > len(partition):
            raise ConfigError(f"requested tile count {t} exceeds partition of {len(partition)}")
    try:
        csv = open(a.out, "w")
    except OSError:
        raise DataError(f"cannot open {a.out} for writing") from None
    rows = []
    with csv:
        csv.write(CSV_HEADER + "\n")
        for w in workers:
            for t in tile_counts:
                res = E.run_offline(ds.frames, cfg, seq, E.RunOptions(iters=a.iters, workers=w, max_tiles=t))
                res.timing.run_id = "bench"
                rows.append(res.timing)
                csv.write(timing_csv_row(res.timing) + "\n")
                csv.flush()
                print(f"workers={w} tiles={t} wall={_fmt(float(res.timing.wall_s))} s")
    for t in tile_counts:
        base = next((r.wall_s for r in rows if r.workers == workers[0] and r.tiles == t), 0.0)
        parts = [f" x{_fmt(base / r.wall_s if r.wall_s > 0 else 0.0)}" for w in workers for r in rows
                 if r.workers == w and r.tiles == t]
        print(f"tiles={t} speedup:" + "".join(parts))
    return 0


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit with the config code (fpm_main.cpp:341-343)
        self.print_usage(sys.stderr)
        print(f"fpm: {message}", file=sys.stderr)
        raise SystemExit(EXIT_CONFIG)


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="fpm", description="parallel Fourier-ptychography reconstruction engine (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    r = sub.add_parser("reconstruct", help="reconstruct HR tiles from a dataset")
    r.add_argument("--data", required=True)
    r.add_argument("--out", required=True)
    r.add_argument("--iters", type=int, default=0)
    r.add_argument("--order", default="")
    r.add_argument("--workers", type=int, default=0)
    r.add_argument("--lag", default="auto")
    r.add_argument("--mode", default="")
    r.add_argument("--online-delay", type=float, default=-1.0)
    r.add_argument("--tiles", type=int, default=0)
    r.add_argument("--unsafe-lag", action="store_true")
    r.add_argument("--force-pipeline", action="store_true")
    r.add_argument("--force", action="store_true")
    r.set_defaults(fn=cmd_reconstruct)
    s = sub.add_parser("stitch", help="stitch HR tiles into one field")
    s.add_argument("--inputs", required=True)
    s.add_argument("--out", required=True)
    s.add_argument("--config", default="")
    s.set_defaults(fn=cmd_stitch)
    e = sub.add_parser("export", help="render amplitude/phase views of a CFI file")
    e.add_argument("--in", dest="input", required=True)
    e.add_argument("--amplitude", default="")
    e.add_argument("--phase", default="")
    e.set_defaults(fn=cmd_export)
    b = sub.add_parser("bench", help="timing sweep over workers and tile counts")
    b.add_argument("--data", required=True)
    b.add_argument("--workers", default="1,2,4,8")
    b.add_argument("--tiles", default="1,4,9,16")
    b.add_argument("--iters", type=int, default=1)
    b.add_argument("--out", required=True)
    b.set_defaults(fn=cmd_bench)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except UnsafeLagError as err:
        print(f"fpm: {err}", file=sys.stderr)
        return EXIT_UNSAFE
    except ConfigError as err:
        print(f"fpm: {err}", file=sys.stderr)
        return EXIT_CONFIG
    except Exception as err:  # DataError, IoError and every other failure (fpm_main.cpp:350-353)
        print(f"fpm: {err}", file=sys.stderr)
        return EXIT_DATA


if __name__ == "__main__":
    sys.exit(main())
