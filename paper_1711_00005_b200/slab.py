"""One large grid over several GPUs: the slab-decomposed march (SURVEY.md
§8(e), BASELINE cfg5).  The reference never splits a frequency's grid; this
is new B200-side capability built on the same kernels.

Per step, the depth sweep runs on azimuth slabs (rank r owns columns
r*Ntheta/N ...), the field is re-distributed by an equal-split all-to-all
(NCCL send/recv over NVLink), the azimuth sweep runs on depth slabs (rank r
owns rows r*Nz/N ...) reading and writing the rank-chunked layout that the
all-to-all delivers, and a second all-to-all returns the next step's
explicit field to the azimuth slabs (C ABI ``pe3d_march_slab``).

* :func:`slab_march` drives N *virtual* ranks from one process on one GPU
  (device copies as the transport) -- the same layouts, kernels and chunk
  bookkeeping as the multi-GPU path, usable and testable on a single B200.
* :func:`distributed_slab_march` is the one-process-per-GPU path: rank 0
  creates the NCCL id, ``torch.distributed`` broadcasts it (plumbing only),
  and each rank marches its slab.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native
from .environment import PERIODIC, gaussian_starter, is_range_independent, wavenumber
from .errors import InvariantError, NativeError
from .marching import _grid_params, _local_column, default_output_stride, steps_within
from .operators import StepCoefficients

NCCL_ID_BYTES = 128


@dataclass
class SlabResult:
    frequency: float
    ranges: np.ndarray
    tl_field: np.ndarray          # [S][Ntheta][Nz] (virtual) or [S][Ntheta][Nz/N] (this rank's slab)
    clamped_samples: int
    final: np.ndarray             # [Ntheta][Nz] or this rank's depth slab [Ntheta][Nz/N]
    step_ms: float                # device time of the step loop
    nranks: int
    rank: Optional[int]


def check_slab_shape(grid, nranks: int) -> None:
    if grid.azimuth_topology != PERIODIC:
        raise InvariantError("slab march: periodic azimuth")
    if nranks < 1 or grid.n_azimuth % nranks:
        raise InvariantError("slab march: n_azimuth % nranks == 0", f"got {grid.n_azimuth} / {nranks}")
    if grid.n_depth % (8 * nranks):
        raise InvariantError("slab march: n_depth % (8 * nranks) == 0", f"got {grid.n_depth} / {nranks}")


def depth_slab(values: np.ndarray, nranks: int, rank: int) -> np.ndarray:
    """Rows of ``values`` [Ntheta][Nz] owned by ``rank`` (contiguous)."""
    nz_s = values.shape[-1] // nranks
    return np.ascontiguousarray(values[..., rank * nz_s:(rank + 1) * nz_s])


def peer_transport_ok(grid, nranks: int) -> bool:
    """Shapes the peer-direct transposes support (pe3d_slab_p2p_export)."""
    nzt = grid.n_depth // 8
    nzt_s = nzt // nranks
    return nranks <= 16 and nzt_s % 32 == 0 and (nzt <= 512 or (nzt % 128 == 0 and nzt // 128 <= 8))


def _run(config, frequency, nranks, rank, nccl_id, n_steps, device, peer_blobs=None):
    grid, env, source, options = config
    check_slab_shape(grid, nranks)
    if not is_range_independent(env):
        raise InvariantError("slab march: range-independent medium")
    k0 = wavenumber(frequency, env.c0)
    coeffs = _native.make_coeffs([k0], [StepCoefficients.for_step(k0, grid.delta_r)])
    steps = steps_within(grid, options.max_range) if n_steps is None else n_steps
    stride = options.output_stride or default_output_stride(grid.n_range)
    S = 1 + steps // stride
    local = _local_column(env, grid, grid.r_start, k0)
    u0 = gaussian_starter(grid, source, k0).values
    virt = nccl_id is None and peer_blobs is None
    if not virt:
        u0 = depth_slab(u0, nranks, rank)
    u0 = np.ascontiguousarray(u0)
    final = np.empty_like(u0)
    tl = np.empty((S,) + u0.shape, dtype=np.float64)
    clamped = np.zeros(1, dtype=np.int64)
    ms = C.c_double(0.0)
    g = _grid_params(grid, 1, steps, stride, 0, grid.r_start)
    if peer_blobs is not None:
        blobs = (C.c_char * len(peer_blobs)).from_buffer_copy(peer_blobs)
        _native.call("pe3d_march_slab_p2p", _native.handle(device), g, coeffs, nranks, rank, blobs,
                     _native.ptr(local), _native.ptr(u0), _native.ptr(final), _native.ptr(tl),
                     _native.ptr(clamped), C.byref(ms))
    else:
        id_buf = None if virt else (C.c_char * NCCL_ID_BYTES).from_buffer_copy(nccl_id)
        _native.call("pe3d_march_slab", _native.handle(device), g, coeffs, nranks, 0 if virt else rank,
                     id_buf, _native.ptr(local), _native.ptr(u0), _native.ptr(final), _native.ptr(tl),
                     _native.ptr(clamped), C.byref(ms))
    ranges = np.asarray([grid.r_start] + [grid.range_at(s * stride) for s in range(1, S)])
    return SlabResult(frequency, ranges, tl, int(clamped[0]), final, ms.value, nranks, None if virt else rank)


def slab_march(config, frequency: float, nranks: int, n_steps: Optional[int] = None,
               device: int = 0) -> SlabResult:
    """Slab-decomposed march with ``nranks`` virtual ranks on one GPU."""
    return _run(config, frequency, nranks, 0, None, n_steps, device)


def new_nccl_id() -> bytes:
    buf = (C.c_char * NCCL_ID_BYTES)()
    status = _native.load_library().pe3d_slab_unique_id(buf, NCCL_ID_BYTES)
    if status != 0:
        raise NativeError("pe3d_slab_unique_id failed (libnccl.so.2 not loadable?)")
    return bytes(buf)


def export_peer_buffers(grid, nranks: int, rank: int, steps: int, stride: int, device: int) -> bytes:
    """Allocate this rank's slab buffers, reset its ordering counters and
    return their CUDA IPC handles (pe3d_slab_p2p_export)."""
    out = (C.c_char * _native.SLAB_IPC_BYTES)()
    g = _grid_params(grid, 1, steps, stride, 0, grid.r_start)
    _native.call("pe3d_slab_p2p_export", _native.handle(device), g, nranks, rank, out)
    return bytes(out)


def distributed_slab_march(config, frequency: float, group=None, device: Optional[int] = None,
                           n_steps: Optional[int] = None, transport: str = "auto") -> SlabResult:
    """One process per GPU: this rank's slab of the decomposed march.

    transport "peer" (the default when the shape allows it): the sweeps store
    their output straight into the other ranks' inputs over NVLink (CUDA IPC
    mappings exchanged here), ordered by device-side counters; "nccl": an
    equal-split all-to-all of NCCL send/recv pairs after each sweep."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = rank if device is None else device
    grid = config.grid
    if transport == "auto":
        transport = "peer" if peer_transport_ok(grid, world) else "nccl"
    if transport == "peer":
        steps = steps_within(grid, config.options.max_range) if n_steps is None else n_steps
        stride = config.options.output_stride or default_output_stride(grid.n_range)
        blob = export_peer_buffers(grid, world, rank, steps, stride, dev)
        blobs = [None] * world
        dist.all_gather_object(blobs, blob, group=group)
        dist.barrier(group=group)                   # every rank's counters reset before anyone marches
        try:
            return _run(config, frequency, world, rank, None, n_steps, dev, peer_blobs=b"".join(blobs))
        finally:
            dist.barrier(group=group)               # no late signal may land in a re-armed counter
    if transport != "nccl":
        raise InvariantError("transport in (auto, peer, nccl)", f"got {transport!r}")
    obj = [new_nccl_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return _run(config, frequency, world, rank, obj[0], n_steps, dev)
