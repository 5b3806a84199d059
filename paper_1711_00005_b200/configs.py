"""The five BASELINE.json configs as in-memory ``Config`` objects.

Synthetic, seeded inputs standing in for the paper's runs; the choices
the BASELINE text leaves open are fixed here and recorded in DESIGN.md §6
(c0 = 1500 m/s, r_start = dr as the reference default ``config.py:202``,
periodic azimuth, output strides, the scaled Munk profile of cfg5, ...).
``n_range``/``frequencies`` may be overridden to cut a config down for
tests while keeping its grid, medium and coefficients.
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

from .config import Config, RunOptions
from .environment import PERIODIC, Absorber, Environment, Grid3D, SoundSpeedProfile, SourceSpec
from .medium import Bathymetry, FluidBottom, LayeredMedium, RandomPerturbation, Sponge

C0 = 1500.0
SPONGE_MAX_ALPHA = 10.0          # dB/lambda at the grid bottom (cfg1 text; reused)
CFG4_NOISE_SEED = 20260814
CFG3_PERTURBATION_SEED = 20260815
CONFIG_NAMES = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")
DEFAULT_STRIDES = {"cfg1": 10, "cfg2": 50, "cfg3": 50, "cfg4": 100, "cfg5": 100}


def munk_speed(z, axis=1300.0, scale=1300.0, c_axis=1500.0, eps=0.00737):
    eta = 2.0 * (np.asarray(z, dtype=np.float64) - axis) / scale
    return c_axis * (1.0 + eps * (eta - 1.0 + np.exp(-eta)))


def _grid(n_range, n_theta, n_depth, dr, dz):
    return Grid3D(n_range=n_range, n_azimuth=n_theta, n_depth=n_depth, delta_r=dr,
                  delta_theta=2.0 * math.pi / n_theta, delta_z=dz, r_start=dr,
                  azimuth_topology=PERIODIC)


def _config(grid, medium, water_depth, freqs, src_depth, stride, n_range_override):
    env = Environment(c0=C0, profile=medium.water, water_depth=water_depth,
                      absorber=Absorber(0.0, 0.0), bottom_depth=grid.depth_extent,
                      medium=medium)
    return Config(grid, env, SourceSpec(frequencies=tuple(freqs), depth=src_depth),
                  RunOptions(output_stride=stride))


def _profile_on_grid(z, c):
    return SoundSpeedProfile(np.asarray(z, dtype=np.float64), np.asarray(c, dtype=np.float64))


def build(name: str, n_range: Optional[int] = None,
          frequencies: Optional[Sequence[float]] = None,
          output_stride: Optional[int] = None) -> Config:
    """Build BASELINE config ``name`` (cfg1..cfg5)."""
    stride = output_stride or DEFAULT_STRIDES[name]
    if name == "cfg1":
        grid = _grid(n_range or 400, 64, 256, 5.0, 1.0)
        medium = LayeredMedium(
            c0=C0, water=SoundSpeedProfile.uniform(1500.0),
            bottom=FluidBottom(1700.0, 1.5, 0.5, Bathymetry(150.0)),
            sponge=Sponge(32, SPONGE_MAX_ALPHA), interface_width=2.0 * grid.delta_z)
        return _config(grid, medium, 150.0, frequencies or (50.0,), 50.0, stride, n_range)
    if name == "cfg2":
        grid = _grid(n_range or 2000, 256, 2048, 10.0, 2.0)
        z = grid.depths()
        medium = LayeredMedium(
            c0=C0, water=_profile_on_grid(z, munk_speed(z)),
            bottom=FluidBottom(1600.0, 1.8, 0.3, Bathymetry(3800.0)),
            sponge=Sponge(128, SPONGE_MAX_ALPHA), interface_width=2.0 * grid.delta_z)
        return _config(grid, medium, 3800.0, frequencies or (100.0,), 1000.0, stride, n_range)
    if name == "cfg3":
        grid = _grid(n_range or 2000, 512, 512, 2.0, 0.5)
        pert = RandomPerturbation(sigma=2.0, corr_h=200.0, corr_v=20.0,
                                  seed=CFG3_PERTURBATION_SEED,
                                  extent_h=2.0 + 2000 * 2.0 + 50.0,   # nominal cfg3 r_max, not n_range

                                  extent_v=grid.depth_extent + 5.0)
        medium = LayeredMedium(
            c0=C0, water=SoundSpeedProfile.uniform(1500.0),
            bottom=FluidBottom(1700.0, 1.5, 0.5, Bathymetry(200.0, 3.0, 5.0)),
            perturbation=pert, interface_width=2.0 * grid.delta_z)
        return _config(grid, medium, 200.0, frequencies or (25.0,), 100.0, stride, n_range)
    if name == "cfg4":
        grid = _grid(n_range or 2000, 256, 1024, 1.0, 0.25)
        z = grid.depths()
        rng = np.random.default_rng(CFG4_NOISE_SEED)
        c = 1520.0 - 0.1 * z + rng.normal(0.0, 0.5, z.size)
        freqs = frequencies or tuple(float(f) for f in np.geomspace(50.0, 500.0, 64))
        medium = LayeredMedium(
            c0=C0, water=_profile_on_grid(z, c),
            bottom=FluidBottom(1650.0, 1.7, 0.4, Bathymetry(200.0)),
            interface_width=2.0 * grid.delta_z)
        return _config(grid, medium, 200.0, freqs, 30.0, stride, n_range)
    if name == "cfg5":
        grid = _grid(n_range or 1000, 4096, 4096, 1.0, 0.5)
        z = grid.depths()
        # "Munk scaled to 0-1800 m": the 0-3800 m Munk column of cfg2 mapped
        # linearly onto 0-1800 m (axis at 1300*1800/3800 m).
        medium = LayeredMedium(
            c0=C0, water=_profile_on_grid(z, munk_speed(z * 3800.0 / 1800.0)),
            bottom=FluidBottom(1600.0, 1.8, 0.3, Bathymetry(1800.0)),
            sponge=Sponge(256, SPONGE_MAX_ALPHA), interface_width=2.0 * grid.delta_z)
        return _config(grid, medium, 1800.0, frequencies or (500.0,), 600.0, stride, n_range)
    raise KeyError(f"unknown config {name!r}; expected one of {CONFIG_NAMES}")
