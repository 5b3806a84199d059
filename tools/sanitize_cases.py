"""Small marches that exercise every sweep kernel, for compute-sanitizer
(racecheck / synccheck / memcheck, one tool per run).  Usage:

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Cases: k_depth_tma + k_azimuth_tma (ring per warp); the split long-column
depth sweep + carry kernel + corrected cluster azimuth sweep; the lock-step
cluster depth sweep (PE3D_DEPTH_NO_SPLIT); the virtual-rank slab march with
peer-direct transposes; the device-medium march; solve_batch.
"""

import math
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1711_00005_b200 import (Absorber, Environment, Grid3D, SoundSpeedProfile, SourceSpec,  # noqa: E402
                                   configs, march_frequencies, slab_march)
from paper_1711_00005_b200.config import Config, RunOptions  # noqa: E402
from paper_1711_00005_b200.tridiag import SolveBatch, solve_batch  # noqa: E402


def cfg_for(n_theta, n_depth, steps=3, freqs=(60.0, 90.0)):
    grid = Grid3D(steps, n_theta, n_depth, 2.0, 2 * math.pi / n_theta, 0.5, 2.0)
    env = Environment(1500.0, SoundSpeedProfile.uniform(1500.0), 6000.0, Absorber(0.8 * grid.depth_extent, 0.01),
                      grid.depth_extent)
    return Config(grid, env, SourceSpec(freqs, 0.3 * grid.depth_extent), RunOptions(output_stride=1))


def main():
    only = sys.argv[1:]
    cases = {
        "warp": lambda: march_frequencies(cfg_for(256, 1024), [60.0, 90.0]),
        "split_cluster": lambda: march_frequencies(cfg_for(1024, 2048, freqs=(60.0,)), [60.0]),
        "nosplit_cluster": lambda: (os.environ.__setitem__("PE3D_DEPTH_NO_SPLIT", "1"),
                                    march_frequencies(cfg_for(1024, 2048, freqs=(60.0,)), [60.0]),
                                    os.environ.pop("PE3D_DEPTH_NO_SPLIT")),
        "slab_peer": lambda: slab_march(cfg_for(256, 2048, freqs=(60.0,)), 60.0, 2),
        "medium": lambda: march_frequencies(configs.build("cfg3", n_range=3, output_stride=1), [25.0]),
        "solve_batch": lambda: solve_batch(SolveBatch(np.full((16, 70), 0.3 + 0.1j), np.full((16, 70), 2.0 + 0j),
                                                      np.full((16, 70), 0.2 - 0.1j),
                                                      np.random.default_rng(0).standard_normal((16, 70)) + 0j,
                                                      "cyclic")),
    }
    for name, fn in cases.items():
        if only and name not in only:
            continue
        fn()
        print("case", name, "ok", flush=True)


if __name__ == "__main__":
    main()
