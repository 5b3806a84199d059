"""Command-line front end: ``python -m paper_1711_00005_b200 run --config X``.

Mirrors the reference's ``pe3d run`` (ref cli.py:37-186): the same flags,
the same precedence for threads/workers (flag > PE3D_THREADS /
PE3D_WORKERS > [run] > 1), the same TL file names and formats, and the
same ``run_manifest.json`` schema -- with every frequency marched on the
GPU (one batched device march) instead of a CPU process farm.  Exit codes:
0 all frequencies ok, 1 some failed, 2 configuration error.

``bench`` runs the GPU micro-benchmarks that replace the reference's
scaling sweep (solve_batch systems/s over the reference's batch sizes, ref
cli.py:34, and march throughput); the invariant selftest of the reference
is not part of this product (out of scope).
"""

from __future__ import annotations

import argparse
import dataclasses
import math
import os
import sys
import time
from pathlib import Path

from . import __version__
from .config import ExecutorSpec, load_config
from .errors import ConfigError, InvariantError, Pe3dError
from .output import file_sha256, tl_filename, write_manifest, write_tl_grid
from .parallel import frequency_farm

ENV_THREADS, ENV_WORKERS = "PE3D_THREADS", "PE3D_WORKERS"
KERNEL_BENCH_BATCHES = (1, 16, 64, 256, 1024)


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1711_00005_b200",
                                description="B200 range march of the 3-D wide-angle PE solver")
    p.add_argument("--version", action="version", version=__version__)
    sub = p.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="march the configured frequencies and write TL grids")
    run.add_argument("--config", required=True)
    run.add_argument("--threads", type=int)
    run.add_argument("--workers", type=int)
    run.add_argument("--output")
    run.add_argument("--stride", type=int)
    run.add_argument("--format", choices=("csv", "binary-grid"), dest="tl_format")
    run.add_argument("--schedule", choices=("static", "dynamic"))
    run.add_argument("--device", type=int, default=0)
    bench = sub.add_parser("bench", help="GPU tridiagonal and march micro-benchmarks")
    bench.add_argument("--config", required=True)
    bench.add_argument("--output")
    return p


def _int_env(name):
    raw = os.environ.get(name)
    if raw is None:
        return None
    try:
        return int(raw)
    except ValueError:
        raise ConfigError(f"environment variable {name}={raw!r} is not an integer") from None


def resolve_executor(options, args) -> ExecutorSpec:
    """flag > environment > [run] section > 1 (ref cli.py:78-90)."""
    threads, workers = options.executor.intra_threads, options.executor.freq_workers
    for env_name, flag, slot in ((ENV_THREADS, "threads", 0), (ENV_WORKERS, "workers", 1)):
        value = _int_env(env_name)
        if getattr(args, flag, None) is not None:
            value = getattr(args, flag)
        if value is not None:
            threads, workers = (value, workers) if slot == 0 else (threads, value)
    return ExecutorSpec(intra_threads=threads, freq_workers=workers)


def _manifest(args, config, executor, entries) -> dict:
    grid, opts = config.grid, config.options
    return {
        "command": "run",
        "package_version": __version__,
        "created_unix": time.time(),
        "config_path": str(Path(args.config).resolve()),
        "config_sha256": file_sha256(args.config),
        "grid": {"n_range": grid.n_range, "n_azimuth": grid.n_azimuth, "n_depth": grid.n_depth,
                 "delta_r_m": grid.delta_r, "delta_theta_deg": math.degrees(grid.delta_theta),
                 "delta_z_m": grid.delta_z, "r_start_m": grid.r_start,
                 "azimuth_topology": grid.azimuth_topology},
        "executor": {"intra_threads": executor.intra_threads, "freq_workers": executor.freq_workers,
                     "schedule": opts.schedule},
        "tl_format": opts.tl_format,
        "frequencies": entries,
    }


def cmd_run(args) -> int:
    try:
        config = load_config(args.config)
        executor = resolve_executor(config.options, args)
        o = config.options
        options = dataclasses.replace(
            o, output_dir=Path(args.output) if args.output else o.output_dir,
            output_stride=o.output_stride if args.stride is None else args.stride,
            tl_format=args.tl_format or o.tl_format, schedule=args.schedule or o.schedule, executor=executor)
    except (ConfigError, InvariantError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 2
    config = config._replace(options=options)
    outdir = options.output_dir
    try:
        outdir.mkdir(parents=True, exist_ok=True)
    except OSError as exc:
        print(f"config error: output_dir not writable: {exc}", file=sys.stderr)
        return 2
    report = frequency_farm(config, config.source.frequencies, workers=executor.freq_workers,
                            schedule=options.schedule, intra_threads=executor.intra_threads, device=args.device)
    entries = []
    for index, frequency in enumerate(config.source.frequencies):
        result = report.results[index]
        if result is None:
            continue
        name = tl_filename(frequency, options.tl_format)
        path = write_tl_grid(outdir / name, result, config.grid, options.tl_format)
        entries.append({"frequency_hz": frequency, "status": "ok", "file": name, "sha256": file_sha256(path),
                        "wall_seconds": result.wall_seconds, "clamped_samples": result.clamped_samples,
                        "output_stride": result.output_stride})
        print(f"frequency {frequency:g} Hz -> {name} ({result.wall_seconds:.2f} s, "
              f"{result.clamped_samples} clamped)")
    for failure in report.failures:
        entries.append({"frequency_hz": failure.frequency, "status": "error", "message": failure.message})
        print(f"frequency {failure.frequency:g} Hz FAILED: {failure.message}", file=sys.stderr)
    write_manifest(outdir, _manifest(args, config, executor, entries))
    return 0 if report.ok else 1


def cmd_bench(args) -> int:
    import numpy as np
    from .tridiag import OPEN, SolveBatch, solve_batch
    try:
        config = load_config(args.config)
    except (ConfigError, InvariantError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 2
    outdir = Path(args.output) if args.output else config.options.output_dir
    outdir.mkdir(parents=True, exist_ok=True)
    rows = ["batch_size,n,seconds,systems_per_second"]
    rng = np.random.default_rng(0)
    n = 128
    for w in KERNEL_BENCH_BATCHES:           # the reference's generator, parallel.py:278-287
        re, im = rng.standard_normal((4, n, w)), rng.standard_normal((4, n, w))
        batch = SolveBatch(0.5 * (re[1, :n - 1] + 1j * im[1, :n - 1]), 4.0 + re[0] + 1j * im[0],
                           0.5 * (re[2, :n - 1] + 1j * im[2, :n - 1]), re[3] + 1j * im[3], OPEN)
        solve_batch(batch)
        t = time.perf_counter()
        solve_batch(batch)
        dt = time.perf_counter() - t
        rows.append(f"{w},{n},{dt:.6f},{w / dt:.1f}")
    (outdir / "kernel_bench.csv").write_text("\n".join(rows) + "\n")
    t = time.perf_counter()
    report = frequency_farm(config, config.source.frequencies)
    wall = time.perf_counter() - t
    g = config.grid
    points = len(config.source.frequencies) * g.n_azimuth * g.n_depth * g.n_range
    summary = "\n".join(rows) + f"\nmarch: {points / wall:.3e} grid-point range-steps/s ({wall:.3f} s, ok={report.ok})\n"
    (outdir / "bench_summary.txt").write_text(summary)
    print(summary, end="")
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return cmd_run(args) if args.command == "run" else cmd_bench(args)
    except Pe3dError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
