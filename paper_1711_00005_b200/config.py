"""Run options and the ``Config`` bundle; ref ``pkg/src/pe3d/config.py:71-102``
and ``ExecutorSpec`` from ``pkg/src/pe3d/pool.py:19-36``.

INI ingestion (ref ``config.py:173-268``) is outside the hot-path scope
(SURVEY.md §8(f) row 4); configs are built in memory, e.g. by
:mod:`.configs`.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path
from typing import NamedTuple, Optional

from .environment import Environment, Grid3D, SourceSpec
from .errors import ConfigError, InvariantError

TL_FORMATS = ("csv", "binary-grid")
SCHEDULES = ("static", "dynamic")
MODES = ("run", "bench", "selftest")
PINNING_MODES = ("none", "compact")


@dataclass(frozen=True)
class ExecutorSpec:
    """Parallelism knobs of the reference.  On the GPU the intra-step
    thread count has no effect (the CUDA grid replaces the thread pool);
    ``freq_workers`` maps to the number of GPUs a farm may use."""

    intra_threads: int = 1
    freq_workers: int = 1
    pinning: str = "none"

    def __post_init__(self):
        if self.intra_threads < 1:
            raise InvariantError("intra_threads >= 1", f"got {self.intra_threads}")
        if self.freq_workers < 1:
            raise InvariantError("freq_workers >= 1", f"got {self.freq_workers}")
        if self.pinning not in PINNING_MODES:
            raise InvariantError(f"pinning in {PINNING_MODES}", f"got {self.pinning!r}")


@dataclass(frozen=True)
class RunOptions:
    mode: str = "run"
    output_dir: Path = Path("out")
    output_stride: Optional[int] = None
    tl_format: str = "csv"
    executor: ExecutorSpec = field(default_factory=ExecutorSpec)
    max_range: Optional[float] = None
    schedule: str = "static"

    def __post_init__(self):
        checks = (
            (self.mode in MODES, f"mode in {MODES}", repr(self.mode)),
            (self.output_stride is None or self.output_stride >= 1,
             "output_stride >= 1", str(self.output_stride)),
            (self.tl_format in TL_FORMATS, f"tl_format in {TL_FORMATS}", repr(self.tl_format)),
            (self.schedule in SCHEDULES, f"schedule in {SCHEDULES}", repr(self.schedule)),
            (self.max_range is None or self.max_range > 0, "max_range > 0", str(self.max_range)),
        )
        for ok, constraint, got in checks:
            if not ok:
                raise InvariantError(constraint, f"got {got}")
        object.__setattr__(self, "output_dir", Path(self.output_dir))


class Config(NamedTuple):
    grid: Grid3D
    environment: Environment
    source: SourceSpec
    options: RunOptions


# ------------------------------------------------------------------ INI files
# Reference schema (ref config.py:1-44, 173-268): [grid] [environment]
# [source] [run], angles in degrees.  Extension: an optional [medium]
# section turns the environment into a LayeredMedium (fluid bottom with
# density and dB/lambda attenuation, bathymetry, absorbing layer, seeded
# perturbation) -- SURVEY.md §8(f) row 4.  Reference files parse unchanged.

def _section_reader(parser, name):
    present = parser.has_section(name)
    sec = parser[name] if present else {}

    def get(key, kind=float, default=None, required=False):
        if key not in sec:
            if required:
                raise ConfigError(f"[{name}] missing required field '{key}'")
            return default
        raw = sec[key]
        if kind is str:
            return raw.strip()
        try:
            return kind(raw)
        except ValueError:
            what = "an integer" if kind is int else "a number"
            raise ConfigError(f"[{name}] field '{key}': expected {what}, got {raw!r}") from None

    get.present = present
    get.has = lambda key: key in sec
    return get


def _profile_from_text(text: str, origin: str):
    import numpy as np
    from .environment import SoundSpeedProfile
    z, c = [], []
    for n, line in enumerate(text.strip().splitlines(), start=1):
        parts = line.replace(",", " ").split()
        if not parts:
            continue
        if len(parts) != 2:
            raise ConfigError(f"{origin}: line {n}: expected 'depth speed', got {line.strip()!r}")
        try:
            z.append(float(parts[0]))
            c.append(float(parts[1]))
        except ValueError:
            raise ConfigError(f"{origin}: line {n}: non-numeric entry in {line.strip()!r}") from None
    if not z:
        raise ConfigError(f"{origin}: empty sound-speed profile")
    return SoundSpeedProfile(np.asarray(z), np.asarray(c))


def load_config(path) -> Config:
    """Parse an INI config (reference schema + optional [medium])."""
    import configparser
    import math
    from .environment import Absorber, Environment, Grid3D, SoundSpeedProfile, SourceSpec

    path = Path(path)
    if not path.exists():
        raise ConfigError(f"config file not found: {path}")
    parser = configparser.ConfigParser(inline_comment_prefixes=("#", ";"))
    try:
        parser.read_string(path.read_text(), source=str(path))
    except configparser.Error as exc:
        raise ConfigError(f"config parse failure: {exc}") from None
    for name in ("grid", "environment", "source"):
        if not parser.has_section(name):
            raise ConfigError(f"missing required section [{name}]")

    g = _section_reader(parser, "grid")
    dr = g("delta_r", required=True)
    grid = Grid3D(n_range=g("n_range", int, required=True), n_azimuth=g("n_azimuth", int, required=True),
                  n_depth=g("n_depth", int, required=True), delta_r=dr,
                  delta_theta=math.radians(g("delta_theta", required=True)), delta_z=g("delta_z", required=True),
                  r_start=g("r_start", default=dr), azimuth_topology=g("azimuth_topology", str, default="periodic"))

    e = _section_reader(parser, "environment")
    if e.has("sound_speed_file"):
        pfile = Path(e("sound_speed_file", str))
        pfile = pfile if pfile.is_absolute() else path.parent / pfile
        if not pfile.exists():
            raise ConfigError(f"sound_speed_file not found: {pfile}")
        profile = _profile_from_text(pfile.read_text(), str(pfile))
    elif e.has("sound_speed_profile"):
        profile = _profile_from_text(e("sound_speed_profile", str), "[environment] sound_speed_profile")
    else:
        profile = SoundSpeedProfile.uniform(e("sound_speed", required=True))
    c0 = e("c0", required=True)
    water_depth = e("water_depth", required=True)
    medium = _medium_from_ini(parser, c0, profile, water_depth, grid)
    env = Environment(c0=c0, profile=profile, water_depth=water_depth,
                      absorber=Absorber(e("absorber_start_depth", default=0.75 * grid.depth_extent),
                                        e("absorber_max_attenuation", default=0.01)),
                      bottom_depth=grid.depth_extent, medium=medium)

    s = _section_reader(parser, "source")
    text = s("frequencies", str, required=True)
    try:
        freqs = tuple(float(tok) for tok in text.split(",") if tok.strip())
    except ValueError:
        raise ConfigError(f"[source] field 'frequencies': expected comma-separated numbers, got {text!r}") from None
    source = SourceSpec(frequencies=freqs, depth=s("depth", required=True), starter=s("starter", str, default="gaussian"))
    if not 0 < source.depth < env.water_depth:
        raise InvariantError("0 < source depth < water_depth",
                             f"got depth {source.depth} vs water_depth {env.water_depth}")

    r = _section_reader(parser, "run")
    options = RunOptions(mode=r("mode", str, default="run"), output_dir=Path(r("output_dir", str, default="out")),
                         output_stride=r("output_stride", int), tl_format=r("tl_format", str, default="csv"),
                         executor=ExecutorSpec(intra_threads=r("threads", int, default=1),
                                               freq_workers=r("workers", int, default=1)),
                         max_range=r("max_range"), schedule=r("schedule", str, default="static"))
    return Config(grid, env, source, options)


def _medium_from_ini(parser, c0, profile, water_depth, grid):
    if not parser.has_section("medium"):
        return None
    from .medium import Bathymetry, FluidBottom, LayeredMedium, RandomPerturbation, Sponge
    m = _section_reader(parser, "medium")
    bathy = Bathymetry(m("bathymetry_depth", default=water_depth), m("bathymetry_slope_deg", default=0.0),
                       m("bathymetry_min_depth", default=0.0))
    bottom = FluidBottom(m("bottom_speed", required=True), m("bottom_density", default=1.0),
                         m("bottom_alpha", default=0.0), bathy)
    n_sponge = m("sponge_points", int, default=0)
    sponge = Sponge(n_sponge, m("sponge_max_alpha", default=10.0)) if n_sponge > 0 else None
    pert = None
    if m.has("perturbation_sigma"):
        pert = RandomPerturbation(sigma=m("perturbation_sigma"), corr_h=m("perturbation_corr_h", required=True),
                                  corr_v=m("perturbation_corr_v", required=True),
                                  seed=m("perturbation_seed", int, required=True),
                                  extent_h=m("perturbation_extent_h", default=grid.max_range + 50.0),
                                  extent_v=m("perturbation_extent_v", default=grid.depth_extent + 5.0))
    return LayeredMedium(c0=c0, water=profile, bottom=bottom, water_density=m("water_density", default=1.0),
                         water_alpha=m("water_alpha", default=0.0), sponge=sponge, perturbation=pert,
                         interface_width=m("interface_width", default=2.0 * grid.delta_z))
