"""ctypes binding of ``libpe3d_b200.so`` (the C ABI in ``include/pe3d_b200.h``).

This is the only way the package computes anything: there is no CPU
fallback.  If the library is missing or no CUDA device is visible, every
compute entry point raises :class:`~.errors.NativeError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path
from typing import Optional

import numpy as np

from .errors import NativeError, raise_from_record

LIB_NAME = "libpe3d_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME
ABI_VERSION = 1

PERIODIC, SECTOR = 0, 1
FLAG_NO_GRAPH, FLAG_SERIAL, FLAG_PROFILE, FLAG_STARTER_COLUMN = 1, 2, 4, 8

# Every symbol include/pe3d_b200.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "pe3d_abi_version", "pe3d_device_count", "pe3d_handle_create", "pe3d_handle_destroy",
    "pe3d_sample_count", "pe3d_march_host", "pe3d_march_device", "pe3d_step_general_host",
    "pe3d_solve_batch_host", "pe3d_profile_last", "pe3d_march_medium_host", "pe3d_slab_unique_id",
    "pe3d_march_slab", "pe3d_slab_p2p_export", "pe3d_march_slab_p2p", "pe3d_last_launches", "pe3d_last_copy_bytes",
    "pe3d_profile_launches", "pe3d_host_alloc", "pe3d_host_free",
)
SLAB_IPC_BYTES = 192


class C128(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class ErrorRecord(C.Structure):
    _fields_ = [("range_index", C.c_int32), ("sweep", C.c_int32), ("member", C.c_int32),
                ("pivot", C.c_int32), ("rank1", C.c_int32), ("frequency", C.c_int32),
                ("message", C.c_char * 208)]


class GridParams(C.Structure):
    _fields_ = [("n_freq", C.c_int32), ("n_theta", C.c_int32), ("n_depth", C.c_int32),
                ("topology", C.c_int32), ("n_steps", C.c_int32), ("output_stride", C.c_int32),
                ("first_index", C.c_int32), ("flags", C.c_int32),
                ("delta_r", C.c_double), ("delta_theta", C.c_double), ("delta_z", C.c_double),
                ("r_start", C.c_double), ("r_input", C.c_double)]


class Coeffs(C.Structure):
    _fields_ = [("k0", C.c_double), ("cx_lhs", C128), ("cx_rhs", C128), ("cy_lhs", C128),
                ("cy_rhs", C128)]


class Medium(C.Structure):
    _fields_ = [("c0", C.c_double), ("n_profile", C.c_int32), ("profile_z", C.c_void_p),
                ("profile_c", C.c_void_p), ("water_density", C.c_double), ("water_alpha", C.c_double),
                ("bottom_speed", C.c_double), ("bottom_density", C.c_double), ("bottom_alpha", C.c_double),
                ("bathy_depth0", C.c_double), ("bathy_slope_deg", C.c_double), ("bathy_min_depth", C.c_double),
                ("sponge_points", C.c_int32), ("sponge_max_alpha", C.c_double),
                ("interface_width", C.c_double), ("lattice", C.c_void_p), ("lat_nx", C.c_int32),
                ("lat_ny", C.c_int32), ("lat_nz", C.c_int32), ("lat_extent_h", C.c_double),
                ("lat_spacing_h", C.c_double), ("lat_spacing_v", C.c_double)]


class Strided(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("row_stride", C.c_int64), ("member_stride", C.c_int64)]


_P = C.c_void_p
_SIGNATURES = {
    "pe3d_abi_version": (C.c_int, []),
    "pe3d_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "pe3d_handle_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p), C.POINTER(ErrorRecord)]),
    "pe3d_handle_destroy": (C.c_int, [_P]),
    "pe3d_sample_count": (C.c_int32, [C.c_int32, C.c_int32]),
    "pe3d_march_host": (C.c_int, [_P, C.POINTER(GridParams), C.POINTER(Coeffs), _P, _P, _P, _P, _P, _P,
                                  C.POINTER(ErrorRecord)]),
    "pe3d_march_device": (C.c_int, [_P, C.POINTER(GridParams), C.POINTER(Coeffs), _P, _P, _P, _P, _P, _P,
                                    _P, C.POINTER(ErrorRecord)]),
    "pe3d_step_general_host": (C.c_int, [_P, C.POINTER(GridParams), C.POINTER(Coeffs), _P, _P, _P, _P,
                                         _P, _P, C.POINTER(ErrorRecord)]),
    "pe3d_solve_batch_host": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, Strided, Strided, Strided,
                                        Strided, _P, C.POINTER(ErrorRecord)]),
    "pe3d_profile_last": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    "pe3d_last_launches": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "pe3d_last_copy_bytes": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pe3d_profile_launches": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_int32)]),
    "pe3d_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "pe3d_host_free": (C.c_int, [_P]),
    "pe3d_march_medium_host": (C.c_int, [_P, C.POINTER(GridParams), C.POINTER(Coeffs), C.POINTER(Medium),
                                         _P, _P, _P, _P, _P, C.POINTER(ErrorRecord)]),
    "pe3d_slab_unique_id": (C.c_int, [_P, C.c_int32]),
    "pe3d_march_slab": (C.c_int, [_P, C.POINTER(GridParams), C.POINTER(Coeffs), C.c_int32, C.c_int32, _P, _P,
                                  _P, _P, _P, _P, C.POINTER(C.c_double), C.POINTER(ErrorRecord)]),
    "pe3d_slab_p2p_export": (C.c_int, [_P, C.POINTER(GridParams), C.c_int32, C.c_int32, _P,
                                       C.POINTER(ErrorRecord)]),
    "pe3d_march_slab_p2p": (C.c_int, [_P, C.POINTER(GridParams), C.POINTER(Coeffs), C.c_int32, C.c_int32, _P, _P,
                                      _P, _P, _P, _P, C.POINTER(C.c_double), C.POINTER(ErrorRecord)]),
}

_lib: Optional[C.CDLL] = None
_lock = threading.Lock()
_handles: dict = {}


def load_library(path: Optional[Path] = None) -> C.CDLL:
    """Load (once) and type the shared library; raises NativeError if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path or os.environ.get("PE3D_B200_LIB", LIB_PATH))
        if not p.exists():
            raise NativeError(f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(or `make -C paper_1711_00005_b200/csrc`); there is no CPU fallback")
        try:
            lib = C.CDLL(str(p))
        except OSError as exc:
            raise NativeError(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.pe3d_abi_version() != ABI_VERSION:
            raise NativeError(f"{p}: ABI version {lib.pe3d_abi_version()} != {ABI_VERSION}")
        if path is None:
            _lib = lib
        return lib


def device_count() -> int:
    n = C.c_int32(0)
    load_library().pe3d_device_count(C.byref(n))
    return int(n.value)


def handle(device: int = 0) -> C.c_void_p:
    """Per-(thread, device) library handle (a handle owns device scratch)."""
    key = (threading.get_ident(), device)
    h = _handles.get(key)
    if h is None:
        lib = load_library()
        if device_count() <= device:
            raise NativeError(f"no CUDA device {device} visible; the B200 path has no CPU fallback")
        h = C.c_void_p()
        err = ErrorRecord()
        raise_from_record(lib.pe3d_handle_create(device, C.byref(h), C.byref(err)), err)
        _handles[key] = h
    return h


def ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    if not a.flags.c_contiguous:
        raise ValueError("native buffers must be C-contiguous")
    return a.ctypes.data_as(C.c_void_p)


def c128(z) -> C128:
    z = complex(z)
    return C128(z.real, z.imag)


def make_coeffs(k0s, coeffs_list) -> "C.Array":
    arr = (Coeffs * len(k0s))()
    for i, (k0, co) in enumerate(zip(k0s, coeffs_list)):
        arr[i] = Coeffs(float(k0), c128(co.cx_lhs), c128(co.cx_rhs), c128(co.cy_lhs), c128(co.cy_rhs))
    return arr


def call(fn_name: str, *args) -> None:
    """Call an ABI entry point and raise the mapped exception on failure."""
    lib = load_library()
    err = ErrorRecord()
    status = getattr(lib, fn_name)(*args, C.byref(err))
    raise_from_record(status, err)


def make_medium(medium, keep_alive: list) -> Medium:
    """pe3d_medium view of a :class:`~.medium.LayeredMedium` (arrays kept
    alive in ``keep_alive`` for the duration of the call)."""
    z = np.ascontiguousarray(medium.water.depths, dtype=np.float64)
    c = np.ascontiguousarray(medium.water.speeds, dtype=np.float64)
    keep_alive += [z, c]
    b = medium.bottom
    m = Medium(c0=medium.c0, n_profile=z.size, profile_z=z.ctypes.data, profile_c=c.ctypes.data,
               water_density=medium.water_density, water_alpha=medium.water_alpha,
               bottom_speed=b.speed, bottom_density=b.density, bottom_alpha=b.alpha,
               bathy_depth0=b.bathymetry.depth0, bathy_slope_deg=b.bathymetry.slope_deg,
               bathy_min_depth=b.bathymetry.min_depth,
               sponge_points=medium.sponge.n_points if medium.sponge else 0,
               sponge_max_alpha=medium.sponge.max_alpha if medium.sponge else 0.0,
               interface_width=medium.interface_width)
    p = medium.perturbation
    if p is not None:
        lat = np.ascontiguousarray(p.lattice, dtype=np.float64)
        keep_alive.append(lat)
        m.lattice = lat.ctypes.data
        m.lat_nx, m.lat_ny, m.lat_nz = lat.shape
        m.lat_extent_h, m.lat_spacing_h, m.lat_spacing_v = p.extent_h, p.spacing_h, p.spacing_v
    return m


# ---------------------------------------------------------------- page-locked host arrays
# The drop-in returns TL stacks and final slabs in page-locked memory, so that
# pe3d_march_host streams the TL samples to the host while the march runs
# (a pageable stack is copied after the march).  Blocks come from
# pe3d_host_alloc; when the last array viewing a block is garbage-collected
# the block returns to a small free list and is reused by the next march
# (page-locking gigabytes costs ~0.1 s/GB, a reused block nothing).

_PINNED_FREE: list = []                # (bytes, ptr) of idle blocks
_pin_lock = threading.RLock()          # a block may be released by the GC inside the pool's own lock
_PINNED_KEEP_BYTES = 24 << 30          # idle blocks kept for reuse (larger ones are released)


class _PinnedBlock:
    """Owner of one page-locked block; numpy arrays over it keep it alive."""

    def __init__(self, ptr: int, nbytes: int, shape, dtype):
        self.ptr, self.nbytes = ptr, nbytes
        self.__array_interface__ = {"shape": tuple(shape), "typestr": np.dtype(dtype).str,
                                    "data": (ptr, False), "version": 3}

    def __del__(self):
        try:
            _pinned_release(self.ptr, self.nbytes)
        except Exception:                  # interpreter shutdown
            pass


def _pinned_release(ptr: int, nbytes: int) -> None:
    with _pin_lock:
        _PINNED_FREE.append((nbytes, ptr))
        _PINNED_FREE.sort()
        while sum(b for b, _ in _PINNED_FREE) > _PINNED_KEEP_BYTES:
            b, p = _PINNED_FREE.pop()
            if _lib is not None:
                _lib.pe3d_host_free(C.c_void_p(p))


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """An uninitialised C-contiguous array in page-locked host memory."""
    nbytes = int(np.prod(shape, dtype=np.int64)) * np.dtype(dtype).itemsize
    if nbytes == 0:
        return np.empty(shape, dtype=dtype)
    lib = load_library()
    ptr = None
    with _pin_lock:
        for i, (b, p) in enumerate(_PINNED_FREE):
            if nbytes <= b <= 2 * nbytes:            # best fit, at most half wasted
                ptr, nbytes_block = p, b
                del _PINNED_FREE[i]
                break
    if ptr is None:
        out = C.c_void_p()
        if lib.pe3d_host_alloc(C.c_uint64(nbytes), C.byref(out)) != 0 or not out.value:
            raise NativeError(f"cannot page-lock {nbytes} bytes of host memory")
        ptr, nbytes_block = out.value, nbytes
    return np.asarray(_PinnedBlock(ptr, nbytes_block, shape, dtype))
