"""Small driver for ncu captures: one cfg4 march of a few steps with the
per-launch profile flag (no graph), so each sweep kernel is a separate,
identifiable launch.  Usage: python tools/profile_march.py [workload] [steps] [r_start]
(r_start: start the march at this range, e.g. 500 for cfg5's split-ring steps)."""

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1711_00005_b200 import _native, configs                  # noqa: E402
from paper_1711_00005_b200.environment import gaussian_starter, wavenumber   # noqa: E402
from paper_1711_00005_b200.marching import _grid_params, _local_column       # noqa: E402
from paper_1711_00005_b200.operators import StepCoefficients                 # noqa: E402


def main():
    import torch
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg = configs.build(name, n_range=max(steps, 3))
    grid, env, source, _ = cfg
    if len(sys.argv) > 3:
        import dataclasses
        grid = dataclasses.replace(grid, r_start=float(sys.argv[3]))
    freqs = list(source.frequencies)
    k0s = [wavenumber(f, env.c0) for f in freqs]
    F, NT, NZ = len(freqs), grid.n_azimuth, grid.n_depth
    coeffs = _native.make_coeffs(k0s, [StepCoefficients.for_step(k, grid.delta_r) for k in k0s])
    local = np.ascontiguousarray(np.stack([_local_column(env, grid, grid.r_start, k) for k in k0s]))
    u0 = np.ascontiguousarray(np.stack([gaussian_starter(grid, source, k).values for k in k0s]))
    dev = torch.device("cuda", 0)
    d_local = torch.from_numpy(local.view(np.float64)).to(dev)
    d_u0 = torch.from_numpy(u0.view(np.float64)).to(dev)
    d_final = torch.empty_like(d_u0)
    tl = torch.empty((F, 1 + steps // steps, NT, NZ), dtype=torch.float64, device=dev)
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
    print({"depth_ms": ms[0] / max(n[0], 1), "azimuth_ms": ms[1] / max(n[1], 1), "other_ms": ms[2], "launches": list(n)})


if __name__ == "__main__":
    main()
