"""Extended ocean medium for the BASELINE configs (NOT in the reference).

The reference's medium is one depth profile plus a quadratic imaginary
ramp (``pkg/src/pe3d/environment.py:234-267``).  The five BASELINE
configs also need a fluid bottom with density and attenuation in dB per
wavelength, a linear absorbing layer, range/azimuth-dependent bathymetry
and a seeded random sound-speed perturbation.
This module is the ONE definition of that medium; the CUDA path, the
checker (``oracle/``) and the golden fixtures (rebinding the reference's
``pe3d.marching.refraction_index_grid``, ref ``marching.py:31,110,116``)
all consume the complex index it returns, so the reference's own march
can serve as the oracle for these media.

Physics choices (recorded in DESIGN.md §6):

* attenuation: n = (c0/c)(1 + i*eta*alpha), eta = 1/(40 pi log10 e),
  alpha in dB/lambda (standard ocean-acoustics convention);
* water/bottom: n^2 blended across the interface z = h(r, theta) by the
  smooth step H = (1 + tanh((z - h)/w))/2, w = ``interface_width``;
* density: the reference's depth operator has a constant off-diagonal
  (ref ``operators.py:231-232``), so density enters only through the local
  term, by the standard transformation p = sqrt(rho) psi:
  n_eff^2 = n^2 + [rho''/(2 rho) - 3/4 (rho'/rho)^2] / k0^2 with rho
  blended by the same H.  This is frequency dependent, hence ``k0``;
* absorbing layer: the last ``n_points`` depth rows get an extra
  attenuation rising linearly to ``max_alpha`` at the grid bottom.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .environment import Grid3D, SoundSpeedProfile
from .errors import DomainError, InvariantError

ETA = 1.0 / (40.0 * math.pi * math.log10(math.e))   # dB/lambda -> Im n / Re n


@dataclass(frozen=True)
class Bathymetry:
    """h(r, theta) = depth0 - r tan(slope) cos(theta), clamped >= min_depth
    (cfg3); ``slope_deg = 0`` gives a flat bottom at ``depth0``."""

    depth0: float
    slope_deg: float = 0.0
    min_depth: float = 0.0

    @property
    def flat(self) -> bool:
        return self.slope_deg == 0.0

    def depth(self, r, theta):
        h = self.depth0 - np.asarray(r) * math.tan(math.radians(self.slope_deg)) * np.cos(theta)
        return np.maximum(h, self.min_depth)


@dataclass(frozen=True)
class FluidBottom:
    speed: float
    density: float
    alpha: float                     # dB per wavelength
    bathymetry: Bathymetry = field(default_factory=lambda: Bathymetry(1e30))


@dataclass(frozen=True)
class Sponge:
    n_points: int
    max_alpha: float                 # dB per wavelength at the grid bottom


@dataclass(frozen=True, eq=False)
class RandomPerturbation:
    """Seeded Gaussian-correlated sound-speed perturbation (cfg3).

    White noise on a Cartesian lattice (x, y horizontal, z vertical) is
    filtered by a separable Gaussian kernel (FFT, periodic) and scaled to
    standard deviation ``sigma``; the medium samples it by trilinear
    interpolation at x = r cos(theta), y = r sin(theta).  The lattice is
    deterministic in ``seed`` and is the data the device path would
    upload, so both sides interpolate the same numbers.
    """

    sigma: float
    corr_h: float
    corr_v: float
    seed: int
    extent_h: float                  # lattice covers [-extent_h, extent_h]^2
    extent_v: float                  # and [0, extent_v] in depth
    lattice: np.ndarray = field(init=False, repr=False)
    spacing_h: float = field(init=False)
    spacing_v: float = field(init=False)

    def __post_init__(self):
        dh, dv = self.corr_h / 4.0, self.corr_v / 4.0
        nx = int(math.ceil(2 * self.extent_h / dh)) + 1
        nz = int(math.ceil(self.extent_v / dv)) + 1
        rng = np.random.default_rng(self.seed)
        noise = rng.standard_normal((nx, nx, nz))
        spectrum = np.fft.rfftn(noise)
        kx = np.fft.fftfreq(nx, d=dh)[:, None, None]
        ky = np.fft.fftfreq(nx, d=dh)[None, :, None]
        kz = np.fft.rfftfreq(nz, d=dv)[None, None, :]
        # Gaussian correlation exp(-d^2/L^2) <-> spectral filter exp(-(pi k L)^2 / 2)
        filt = np.exp(-0.5 * (math.pi ** 2) * ((kx * self.corr_h) ** 2 + (ky * self.corr_h) ** 2
                                                + (kz * self.corr_v) ** 2))
        field_ = np.fft.irfftn(spectrum * filt, s=noise.shape, axes=(0, 1, 2))
        field_ *= self.sigma / field_.std()
        object.__setattr__(self, "lattice", np.ascontiguousarray(field_))
        object.__setattr__(self, "spacing_h", dh)
        object.__setattr__(self, "spacing_v", dv)

    def sample(self, x, y, z):
        """Trilinear interpolation of the lattice (clamped at its edges)."""
        lat = self.lattice
        fx = np.clip((np.asarray(x) + self.extent_h) / self.spacing_h, 0, lat.shape[0] - 1.000001)
        fy = np.clip((np.asarray(y) + self.extent_h) / self.spacing_h, 0, lat.shape[1] - 1.000001)
        fz = np.clip(np.asarray(z) / self.spacing_v, 0, lat.shape[2] - 1.000001)
        ix, iy, iz = fx.astype(np.int64), fy.astype(np.int64), fz.astype(np.int64)
        tx, ty, tz = fx - ix, fy - iy, fz - iz
        out = 0.0
        for ox, wx in ((0, 1 - tx), (1, tx)):
            for oy, wy in ((0, 1 - ty), (1, ty)):
                for oz, wz in ((0, 1 - tz), (1, tz)):
                    out = out + wx * wy * wz * lat[ix + ox, iy + oy, iz + oz]
        return out


@dataclass(frozen=True, eq=False)
class LayeredMedium:
    """Water column over a fluid bottom, with optional absorbing layer,
    bathymetry and perturbation.  See the module docstring for the model.
    """

    c0: float
    water: SoundSpeedProfile
    bottom: FluidBottom
    water_density: float = 1.0
    water_alpha: float = 0.0
    sponge: Optional[Sponge] = None
    perturbation: Optional[RandomPerturbation] = None
    interface_width: float = 1.0     # metres; smoothing of the water/bottom step

    def __post_init__(self):
        if not self.interface_width > 0:
            raise InvariantError("interface_width > 0")
        if self.sponge is not None and self.sponge.n_points < 1:
            raise InvariantError("sponge.n_points >= 1")

    @property
    def range_independent(self) -> bool:
        return self.bottom.bathymetry.flat and self.perturbation is None

    @property
    def has_density_contrast(self) -> bool:
        return self.bottom.density != self.water_density

    def _sponge_alpha(self, grid: Grid3D) -> np.ndarray:
        alpha = np.zeros(grid.n_depth)
        if self.sponge is not None:
            n = min(self.sponge.n_points, grid.n_depth)
            alpha[grid.n_depth - n:] = self.sponge.max_alpha * np.arange(1, n + 1) / n
        return alpha

    def index_squared(self, grid: Grid3D, r: float, theta, k0: Optional[float]) -> np.ndarray:
        """n_eff^2 at range r for the azimuths ``theta`` (array), shape
        (len(theta), n_depth)."""
        if self.has_density_contrast and k0 is None:
            raise DomainError("a medium with a density contrast needs k0")
        theta = np.atleast_1d(np.asarray(theta, dtype=np.float64))[:, None]
        z = grid.depths()[None, :]
        c_w = self.water.speed_at(grid.depths())[None, :]
        if self.perturbation is not None:
            c_w = c_w + self.perturbation.sample(r * np.cos(theta), r * np.sin(theta), z)
        n2_w = ((self.c0 / c_w) * (1.0 + 1j * ETA * self.water_alpha)) ** 2
        b = self.bottom
        n2_b = ((self.c0 / b.speed) * (1.0 + 1j * ETA * b.alpha)) ** 2
        h = b.bathymetry.depth(r, theta)
        w = self.interface_width
        t = np.tanh((z - h) / w)
        step = 0.5 * (1.0 + t)
        n2 = (1.0 - step) * n2_w + step * n2_b
        n2 = n2 * (1.0 + 1j * ETA * self._sponge_alpha(grid)[None, :]) ** 2
        if self.has_density_contrast:
            jump = b.density - self.water_density
            sech2 = 1.0 - t * t
            rho = self.water_density + jump * step
            d1 = jump * sech2 / (2.0 * w)
            d2 = -jump * sech2 * t / (w * w)
            n2 = n2 + (d2 / (2.0 * rho) - 0.75 * (d1 / rho) ** 2) / (k0 * k0)
        return n2

    def _column_parts(self, grid: Grid3D):
        """Range-independent media: the k0-independent n^2 column and the
        density term's numerator, computed once per depth grid (a batch of
        frequencies shares them; index_squared's arithmetic, term by term)."""
        key = (grid.n_depth, grid.delta_z)
        cache = self.__dict__.setdefault("_parts_cache", {})
        parts = cache.get(key)
        if parts is None:
            z = grid.depths()[None, :]
            c_w = self.water.speed_at(grid.depths())[None, :]
            n2_w = ((self.c0 / c_w) * (1.0 + 1j * ETA * self.water_alpha)) ** 2
            b = self.bottom
            n2_b = ((self.c0 / b.speed) * (1.0 + 1j * ETA * b.alpha)) ** 2
            h = b.bathymetry.depth(0.0, np.zeros((1, 1)))
            w = self.interface_width
            t = np.tanh((z - h) / w)
            step = 0.5 * (1.0 + t)
            n2 = (1.0 - step) * n2_w + step * n2_b
            n2 = n2 * (1.0 + 1j * ETA * self._sponge_alpha(grid)[None, :]) ** 2
            dens = None
            if self.has_density_contrast:
                jump = b.density - self.water_density
                sech2 = 1.0 - t * t
                rho = self.water_density + jump * step
                d1 = jump * sech2 / (2.0 * w)
                d2 = -jump * sech2 * t / (w * w)
                dens = d2 / (2.0 * rho) - 0.75 * (d1 / rho) ** 2
            parts = cache[key] = (n2, dens)
        return parts

    def index_grid(self, grid: Grid3D, r: float, k0: Optional[float]) -> np.ndarray:
        """Complex n (principal square root of n_eff^2), (n_azimuth, n_depth)."""
        if self.range_independent:
            if self.has_density_contrast and k0 is None:
                raise DomainError("a medium with a density contrast needs k0")
            n2, dens = self._column_parts(grid)
            if dens is not None:
                n2 = n2 + dens / (k0 * k0)
            column = np.sqrt(n2[0])
            return np.broadcast_to(column, (grid.n_azimuth, grid.n_depth))
        return np.sqrt(self.index_squared(grid, r, grid.azimuths(), k0))
