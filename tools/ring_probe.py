"""Sweep time per launch vs ring length at a fixed field size (HBM-sized):
cfg4's medium and 64 frequencies with the grid reshaped to n_theta x n_depth
(n_theta * n_depth = 256 * 1024), so the azimuth sweep runs the ring-per-warp
kernel (n_theta <= 512) or the cluster kernel with 2/4/8 segments.

    python tools/ring_probe.py [steps]"""
import ctypes as C
import dataclasses
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1711_00005_b200 import _native, configs                  # noqa: E402
from paper_1711_00005_b200.environment import gaussian_starter, wavenumber   # noqa: E402
from paper_1711_00005_b200.marching import _grid_params, _local_column       # noqa: E402
from paper_1711_00005_b200.operators import StepCoefficients                 # noqa: E402


def probe(n_theta, n_depth, steps):
    import torch
    cfg = configs.build("cfg4", n_range=max(steps, 3))
    grid, env, source, opts = cfg
    grid = dataclasses.replace(grid, n_azimuth=n_theta, n_depth=n_depth, delta_theta=2 * math.pi / n_theta)
    freqs = list(source.frequencies)
    k0s = [wavenumber(f, env.c0) for f in freqs]
    F = len(freqs)
    coeffs = _native.make_coeffs(k0s, [StepCoefficients.for_step(k, grid.delta_r) for k in k0s])
    local = np.ascontiguousarray(np.stack([_local_column(env, grid, grid.r_start, k) for k in k0s]))
    src = dataclasses.replace(source, depth=min(source.depth, 0.5 * grid.depth_extent))
    u0 = np.ascontiguousarray(np.stack([gaussian_starter(grid, src, k).values for k in k0s]))
    dev = torch.device("cuda", 0)
    d_local = torch.from_numpy(local.view(np.float64)).to(dev)
    d_u0 = torch.from_numpy(u0.view(np.float64)).to(dev)
    d_final = torch.empty_like(d_u0)
    tl = torch.empty((F, 2, n_theta, n_depth), dtype=torch.float64, device=dev)
    cl = torch.zeros(F, dtype=torch.int64, device=dev)
    g = _grid_params(grid, F, steps, steps, 0, grid.r_start, _native.FLAG_PROFILE)
    h = _native.handle(0)
    for _ in range(2):
        _native.call("pe3d_march_device", h, g, coeffs, C.c_void_p(d_local.data_ptr()), C.c_void_p(d_u0.data_ptr()),
                     C.c_void_p(d_final.data_ptr()), C.c_void_p(tl.data_ptr()), None, C.c_void_p(cl.data_ptr()), None)
    torch.cuda.synchronize()
    ms = (C.c_double * 3)()
    n = (C.c_int32 * 3)()
    _native.load_library().pe3d_profile_last(h, ms, n)
    k1, k2 = ms[0] / max(n[0], 1), ms[1] / max(n[1], 1)
    gb = 32 * F * n_theta * n_depth / 1e9
    print(f"n_theta {n_theta:5d} n_depth {n_depth:5d}: depth {k1 * 1e3:7.1f} us ({gb / k1:.0f} GB/s)  "
          f"azimuth {k2 * 1e3:7.1f} us ({gb / k2:.0f} GB/s)", flush=True)


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    for nt, nz in ((256, 1024), (512, 512), (1024, 256), (2048, 128), (4096, 64)):
        probe(nt, nz, steps)
