"""Range marching on the B200: the drop-in for ``pkg/src/pe3d/marching.py``.

``run_frequency`` (ref :144-193) and ``range_step`` (ref :93-136) keep the
reference's signatures, state objects, results and exceptions; the
arithmetic of every step runs in the sm_100a kernels of ``csrc/`` through
the C ABI (``libpe3d_b200.so``).  ``march_frequencies`` is the batched
entry point: many frequencies of one config in one device march (the body
of ``frequency_farm``).

* Range-independent media (every reference ``Environment``, and extended
  media without bathymetry slope or perturbation): ``pe3d_march_host``,
  the depth matrix factored once per frequency on the device and the step
  loop one CUDA graph (concurrent frequency chains).
* Range/azimuth-dependent ``LayeredMedium`` (cfg3): ``pe3d_march_medium_host``,
  the medium regenerated on the device every step.
* Any other range-dependent environment: one range step per ABI call
  (``pe3d_step_general_host``) with the per-point local term of both ranges
  computed on the host, as the reference does.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _native
from .environment import (
    PERIODIC, SECTOR, Environment, FieldSlab, Grid3D, gaussian_starter, gaussian_starter_column,
    is_range_independent, local_term_grid, refraction_index_grid, wavenumber,
)
from .errors import DomainError
from .operators import StepCoefficients

MAX_OUTPUT_SAMPLES = 512   # ref marching.py:45
# Device memory budget for one batched march (TL stack dominates), bytes.
BATCH_BYTES = 48 << 30


@dataclass(eq=False)
class MarchState:
    """ref marching.py:48-62."""

    slab: FieldSlab
    range_index: int
    coeffs: StepCoefficients
    environment: Environment
    grid: Grid3D
    k0: float
    intra_threads: int = 1


@dataclass(eq=False)
class FrequencyResult:
    """ref marching.py:65-77 (plus optional field snapshots at the TL ranges)."""

    frequency: float
    ranges: np.ndarray
    tl_field: np.ndarray
    clamped_samples: int
    final_slab: FieldSlab
    output_stride: int
    wall_seconds: float
    snapshots: Optional[np.ndarray] = None


def apply_boundary(slab: FieldSlab, grid: Grid3D, env: Environment) -> FieldSlab:
    """Zero the surface row (and sector edges) of a host slab in place;
    ref marching.py:80-90.  (On the device the same rule is fused into the
    kernels.)"""
    slab.check_grid(grid)
    slab.values[:, 0] = 0.0
    if grid.azimuth_topology == SECTOR:
        slab.values[0, :] = 0.0
        slab.values[-1, :] = 0.0
    return slab


def default_output_stride(n_steps: int) -> int:
    """ref marching.py:139-141."""
    return max(1, (n_steps + 1 + MAX_OUTPUT_SAMPLES - 1) // MAX_OUTPUT_SAMPLES)


def steps_within(grid: Grid3D, max_range: Optional[float]) -> int:
    """Number of steps run_frequency takes (the max_range cut with 1e-12
    slack, ref marching.py:177-179)."""
    if max_range is None:
        return grid.n_range
    n = 0
    for j in range(1, grid.n_range + 1):
        if grid.range_at(j) > max_range * (1.0 + 1e-12):
            break
        n = j
    return n


def _grid_params(grid: Grid3D, n_freq: int, n_steps: int, stride: int, first_index: int,
                 r_input: float, flags: int = 0) -> _native.GridParams:
    return _native.GridParams(
        n_freq, grid.n_azimuth, grid.n_depth,
        _native.PERIODIC if grid.azimuth_topology == PERIODIC else _native.SECTOR,
        n_steps, stride, first_index, flags,
        grid.delta_r, grid.delta_theta, grid.delta_z, grid.r_start, r_input)


def _device_medium(env) -> bool:
    """The medium can be generated on the device (a LayeredMedium)."""
    from .medium import LayeredMedium
    return isinstance(getattr(env, "medium", None), LayeredMedium)


def _local_column(env, grid: Grid3D, r: float, k0: float) -> np.ndarray:
    """n^2 - 1 over depth for a range-independent medium (the same
    elementwise arithmetic as local_term_grid, ref operators.py:93, on one
    column of the azimuth-independent index grid)."""
    n = np.asarray(refraction_index_grid(env, grid, r, k0)[0], dtype=np.complex128)
    return np.ascontiguousarray(n ** 2 - 1.0)


def _local_columns(env, grid: Grid3D, r: float, k0s) -> np.ndarray:
    """_local_column of every frequency, [F][n_depth].  A range-independent
    LayeredMedium evaluates its k0-independent column once and adds the density
    term per frequency in one array expression (elementwise the same
    arithmetic as index_grid, so the same bits)."""
    from .medium import LayeredMedium
    medium = getattr(env, "medium", None)
    if isinstance(medium, LayeredMedium) and medium.range_independent and len(k0s) > 1:
        # the last batch's columns are kept with the medium, next to its k0-independent
        # parts (a farm called again on the same frequencies: 1 ms of complex square roots
        # of a 20-step cfg4 march's 8 ms); read-only, the march only uploads them
        key = (grid.n_depth, grid.delta_z, tuple(k0s))
        kept = medium.__dict__.get("_local_columns_cache")
        if kept is not None and kept[0] == key:
            return kept[1]
        n2, dens = medium._column_parts(grid)
        n2 = np.broadcast_to(n2[0], (len(k0s), grid.n_depth))
        if dens is not None:
            k0 = np.asarray(k0s, dtype=np.float64)[:, None]
            n2 = n2 + dens[0][None, :] / (k0 * k0)
        cols = np.ascontiguousarray(np.sqrt(n2) ** 2 - 1.0)
        cols.setflags(write=False)
        medium.__dict__["_local_columns_cache"] = (key, cols)
        return cols
    return np.ascontiguousarray(np.stack([_local_column(env, grid, r, k0) for k0 in k0s]))


def _starter_columns(grid: Grid3D, source, k0s) -> np.ndarray:
    """The Gaussian starter of every frequency as one depth column each
    (azimuth independent, surface zero; ref environment.py:270-284) -- the
    march reads them with PE3D_FLAG_STARTER_COLUMN.  One array expression
    for all frequencies: elementwise the arithmetic of gaussian_starter_column."""
    if len(k0s) == 0:
        return np.empty((0, grid.n_depth), dtype=np.complex128)
    gaussian_starter_column(grid, source, k0s[0])              # validates the source depth
    z = grid.depths()
    k0 = np.asarray(k0s, dtype=np.float64)[:, None]
    cols = (np.sqrt(k0) * np.exp(-0.5 * k0 * k0 * (z - source.depth) ** 2)).astype(np.complex128)
    cols[:, 0] = 0.0
    return np.ascontiguousarray(cols)


def range_step(state: MarchState, device: int = 0) -> MarchState:
    """Advance one range step on the GPU; ref marching.py:93-136."""
    grid = state.grid
    j = state.range_index
    if j + 1 > grid.n_range:
        raise DomainError(f"step {j + 1} exceeds n_range {grid.n_range}")
    slab = state.slab
    apply_boundary(slab, grid, state.environment)
    if state.coeffs.delta == 0:
        # identity step, returned to the bit (ref marching.py:102-107)
        return MarchState(slab, j + 1, state.coeffs, state.environment, grid, state.k0,
                          state.intra_threads)
    r_new = grid.range_at(j + 1)
    env, k0 = state.environment, state.k0
    coeffs = _native.make_coeffs([k0], [state.coeffs])
    u_in = np.ascontiguousarray(slab.values, dtype=np.complex128)
    u_out = np.empty_like(u_in)
    h = _native.handle(device)
    if is_range_independent(env):
        local = _local_column(env, grid, slab.range_m, k0)
        g = _grid_params(grid, 1, 1, 1, j, slab.range_m)
        _native.call("pe3d_march_host", h, g, coeffs, _native.ptr(local), _native.ptr(u_in),
                     _native.ptr(u_out), None, None, None)
    elif _device_medium(env):
        keep: list = []
        g = _grid_params(grid, 1, 1, 1, j, slab.range_m)
        _native.call("pe3d_march_medium_host", h, g, coeffs, _native.make_medium(env.medium, keep),
                     _native.ptr(u_in), _native.ptr(u_out), None, None, None)
    else:
        now = np.ascontiguousarray(local_term_grid(env, grid, slab.range_m, k0))
        new = np.ascontiguousarray(local_term_grid(env, grid, r_new, k0))
        g = _grid_params(grid, 1, 1, 1, j, slab.range_m)
        _native.call("pe3d_step_general_host", h, g, coeffs, _native.ptr(now), _native.ptr(new),
                     _native.ptr(u_in), _native.ptr(u_out), None, None)
    return MarchState(FieldSlab(u_out, r_new), j + 1, state.coeffs, env, grid, k0,
                      state.intra_threads)


def _freq_setup(config, frequencies):
    grid, env, source, options = config
    for f in frequencies:
        if f not in source.frequencies:
            raise DomainError(f"frequency {f} is not one of the source frequencies")
    k0s = [wavenumber(f, env.c0) for f in frequencies]
    coeffs = [StepCoefficients.for_step(k0, grid.delta_r) for k0 in k0s]
    return k0s, coeffs


def march_frequencies(config, frequencies: Sequence[float], n_steps: Optional[int] = None,
                      keep_snapshots: bool = False, device: int = 0,
                      flags: int = 0) -> List[FrequencyResult]:
    """March several frequencies of one config as one device batch.

    Returns one FrequencyResult per frequency, in order.  Raises the
    reference's StepError for the lowest failing frequency; use
    :func:`~.parallel.frequency_farm` for per-frequency failure isolation.
    """
    t0 = time.perf_counter()
    grid, env, source, options = config
    frequencies = [float(f) for f in frequencies]
    k0s, coeffs = _freq_setup(config, frequencies)
    steps = steps_within(grid, options.max_range) if n_steps is None else n_steps
    stride = options.output_stride or default_output_stride(grid.n_range)
    S = 1 + steps // stride
    ranges = np.asarray([grid.r_start] + [grid.range_at(s * stride) for s in range(1, S)])
    F, NT, NZ = len(frequencies), grid.n_azimuth, grid.n_depth
    slab_elems = NT * NZ

    # TL stack and final slabs in page-locked memory: the TL samples stream to
    # the host while the march runs (pe3d_march_host)
    tl = _native.pinned_empty((F, S, NT, NZ), np.float64)
    snaps = np.empty((F, S, NT, NZ), dtype=np.complex128) if keep_snapshots else None
    final = _native.pinned_empty((F, NT, NZ), np.complex128)
    clamped = np.zeros(F, dtype=np.int64)
    h = _native.handle(device)

    if is_range_independent(env):
        cols = _starter_columns(grid, source, k0s)
        per_freq = slab_elems * (S * (8 + (16 if keep_snapshots else 0)) + 16 * 6)
        chunk = max(1, min(F, BATCH_BYTES // max(per_freq, 1)))
        for lo in range(0, F, chunk):
            hi = min(F, lo + chunk)
            local = _local_columns(env, grid, grid.r_start, k0s[lo:hi])
            g = _grid_params(grid, hi - lo, steps, stride, 0, grid.r_start, flags | _native.FLAG_STARTER_COLUMN)
            cf = _native.make_coeffs(k0s[lo:hi], coeffs[lo:hi])
            _native.call("pe3d_march_host", h, g, cf, _native.ptr(local), _native.ptr(cols[lo:hi]),
                         _native.ptr(final[lo:hi]), _native.ptr(tl[lo:hi]),
                         _native.ptr(snaps[lo:hi]) if keep_snapshots else None,
                         _native.ptr(clamped[lo:hi]))
    elif _device_medium(env):
        keep: list = []
        med = _native.make_medium(env.medium, keep)
        g = _grid_params(grid, F, steps, stride, 0, grid.r_start, flags | _native.FLAG_STARTER_COLUMN)
        cf = _native.make_coeffs(k0s, coeffs)
        _native.call("pe3d_march_medium_host", h, g, cf, med, _native.ptr(_starter_columns(grid, source, k0s)),
                     _native.ptr(final),
                     _native.ptr(tl), _native.ptr(snaps) if keep_snapshots else None, _native.ptr(clamped))
    else:
        u0 = np.empty((F, NT, NZ), dtype=np.complex128)
        for i, k0 in enumerate(k0s):
            u0[i] = gaussian_starter(grid, source, k0).values
        _march_general(config, k0s, coeffs, u0, steps, stride, tl, snaps, final, clamped, h)

    wall = time.perf_counter() - t0
    r_final = grid.range_at(steps) if steps else grid.r_start
    return [FrequencyResult(frequency=frequencies[i], ranges=ranges.copy(), tl_field=tl[i],
                            clamped_samples=int(clamped[i]),
                            final_slab=FieldSlab(final[i], r_final), output_stride=stride,
                            wall_seconds=wall, snapshots=None if snaps is None else snaps[i])
            for i in range(F)]


def _march_general(config, k0s, coeffs, u0, steps, stride, tl, snaps, final, clamped, h):
    """Range/azimuth-dependent media: one ABI step per range step, TL of the
    recorded steps computed on the device."""
    grid, env, _, _ = config
    F = len(k0s)
    cf = _native.make_coeffs(k0s, coeffs)
    u = np.ascontiguousarray(u0.copy())
    u[:, :, 0] = 0.0
    if grid.azimuth_topology == SECTOR:
        u[:, 0, :] = 0.0
        u[:, -1, :] = 0.0
    # sample 0: TL of the starter via a zero-step device march on a flat medium
    g0 = _grid_params(grid, F, 0, stride, 0, grid.r_start)
    zero_local = np.zeros((F, grid.n_depth), dtype=np.complex128)
    tl0 = np.empty((F, 1) + u.shape[1:], dtype=np.float64)
    c0 = np.zeros(F, dtype=np.int64)
    _native.call("pe3d_march_host", h, g0, cf, _native.ptr(zero_local), _native.ptr(u), None,
                 _native.ptr(tl0), None, _native.ptr(c0))
    tl[:, 0] = tl0[:, 0]
    clamped += c0
    if snaps is not None:
        snaps[:, 0] = u
    final[:] = u
    tl_step = np.empty((F,) + u.shape[1:], dtype=np.float64)
    c_step = np.zeros(F, dtype=np.int64)
    r = grid.r_start
    for s in range(steps):
        r_new = grid.range_at(s + 1)
        now = np.ascontiguousarray(np.stack([local_term_grid(env, grid, r, k0) for k0 in k0s]))
        new = np.ascontiguousarray(np.stack([local_term_grid(env, grid, r_new, k0) for k0 in k0s]))
        out = np.empty_like(u)
        record = (s + 1) % stride == 0
        g = _grid_params(grid, F, 1, 1, s, r)
        _native.call("pe3d_step_general_host", h, g, cf, _native.ptr(now), _native.ptr(new),
                     _native.ptr(u), _native.ptr(out), _native.ptr(tl_step) if record else None,
                     _native.ptr(c_step) if record else None)
        u, r = out, r_new
        if record:
            k = (s + 1) // stride
            tl[:, k] = tl_step
            clamped += c_step
            if snaps is not None:
                snaps[:, k] = u
    final[:] = u


def run_frequency(config, frequency: float, executor=None, device: int = 0) -> FrequencyResult:
    """March one frequency from the starter range to max range on the GPU;
    ref marching.py:144-193 (same TL sampling, stride default, max_range
    cut, result fields).  ``executor`` is accepted for signature
    compatibility (the GPU grid replaces intra-step threads)."""
    return march_frequencies(config, [frequency], device=device)[0]
