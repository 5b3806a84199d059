"""Full-length golden fixtures for BASELINE cfg2-cfg5, made by running the
REFERENCE package itself over every range step of each config.

Run in the build container (where /root/reference exists), one config per
process (they are long: about 9 / 6 / 45 min and 3 h on this host):

    python tests/golden/make_full_length.py cfg2
    python tests/golden/make_full_length.py cfg4 --workers 6

Single-frequency configs go through the reference's ``run_frequency``
(ref marching.py:144-193); cfg4's 64 frequencies go through the
reference's ``frequency_farm`` (ref parallel.py:143-185) with worker
processes.  The BASELINE media, which the reference cannot express, are
injected by rebinding ``pe3d.marching.refraction_index_grid`` (ref
marching.py:31,110,116) to the shared medium of
``paper_1711_00005_b200.medium``; everything else (operators, assembly,
Thomas / Sherman-Morrison, boundary, TL) is the reference's own code.

``pe3d.marching.range_step`` is wrapped (the wrapper calls the original
and looks at its result) so that, at every output range j % stride == 0
(ref marching.py:181-183), the field is sampled at SAMPLE_POINTS seeded
(theta, depth) points and its full-grid L2 norm is recorded.  From the
returned ``FrequencyResult`` the fixture keeps, at every output range:
TL at the same points (float64), the whole theta-0 TL column, and two
whole-grid TL statistics (the count of samples with TL < 150 dB and the
sum of those TL values).  Plus the ranges, clamped count, and the final
slab at the points and on the theta-0 column.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, os.environ.get("PE3D_REFERENCE_SRC", "/root/reference/pkg/src"))

import pe3d                                      # noqa: E402  (the reference)
import pe3d.marching as ref_marching             # noqa: E402

from paper_1711_00005_b200 import configs        # noqa: E402
from paper_1711_00005_b200.environment import refraction_index_grid  # noqa: E402

SAMPLE_POINTS = {"cfg2": 512, "cfg3": 512, "cfg4": 128, "cfg5": 512}
TL_CUT = 150.0
SEED = 5151

_CFG = {}           # per process: the product-side config whose medium is injected
_ORIG_STEP = ref_marching.range_step
_REC_DIR = None


def ref_grid(g):
    return pe3d.Grid3D(g.n_range, g.n_azimuth, g.n_depth, g.delta_r, g.delta_theta,
                       g.delta_z, g.r_start, g.azimuth_topology)


def ref_env(g, c0=1500.0):
    return pe3d.Environment(c0, pe3d.SoundSpeedProfile.uniform(c0), 6000.0,
                            pe3d.Absorber(0.0, 0.0), g.depth_extent)


def sample_points(name, g):
    rng = np.random.default_rng(SEED)
    n = SAMPLE_POINTS[name]
    return rng.integers(0, g.n_azimuth, n), rng.integers(0, g.n_depth, n)


def _recording_step(state):
    """Reference range_step, then record the sampled field at output ranges."""
    cfg = _CFG["cfg"]
    _CFG["k0"] = state.k0               # the injected n-grid needs this step's k0 (density term)
    new = _ORIG_STEP(state)
    j = new.range_index
    if j % _CFG["stride"] == 0:
        u = new.slab.values
        rec = _CFG["rec"].setdefault(state.k0, ([], []))
        rec[0].append(u[_CFG["mi"], _CFG["li"]].copy())
        rec[1].append(float(np.linalg.norm(u)))
        if _REC_DIR is not None and j == cfg.grid.n_range:
            np.savez(Path(_REC_DIR) / f"rec_{state.k0!r}.npz", k0=state.k0,
                     samples=np.stack(rec[0]), norms=np.array(rec[1]))
    return new


def install(name, cfg, rec_dir=None):
    """Bind the shared medium and the recording wrapper into the reference."""
    global _REC_DIR
    g, env = cfg.grid, cfg.environment
    mi, li = sample_points(name, g)
    _CFG.update(cfg=cfg, stride=cfg.options.output_stride, mi=mi, li=li, rec={}, k0=None)
    _REC_DIR = rec_dir
    ref_marching.refraction_index_grid = lambda e, gg, r: refraction_index_grid(env, g, r, _CFG["k0"])
    ref_marching.range_step = _recording_step


def ref_config(cfg, freqs):
    g = cfg.grid
    return pe3d.Config(ref_grid(g), ref_env(g), pe3d.SourceSpec(tuple(freqs), cfg.source.depth),
                       pe3d.RunOptions(output_stride=cfg.options.output_stride))


def tl_record(res, mi, li, col_dtype):
    tl = res.tl_field
    below = tl < TL_CUT
    return dict(ranges=res.ranges, tl_points=tl[:, mi, li].copy(),
                tl_col0=tl[:, 0, :].astype(col_dtype),
                tl_count=below.sum(axis=(1, 2)).astype(np.int64),
                tl_sum=np.where(below, tl, 0.0).sum(axis=(1, 2)),
                clamped=res.clamped_samples,
                final_points=res.final_slab.values[mi, li].copy(),
                final_col0=res.final_slab.values[0].copy())


def single(name, threads=1):
    cfg = configs.build(name)
    f = cfg.source.frequencies[0]
    install(name, cfg)
    from paper_1711_00005_b200.environment import wavenumber
    _CFG["k0"] = wavenumber(f, cfg.environment.c0)
    t0 = time.perf_counter()
    # intra_threads only splits the reference's fixed 64-member tiles across
    # threads; its output does not depend on it (ref tridiag.py:248-255).
    res = pe3d.run_frequency(ref_config(cfg, (f,)), f, pe3d.ExecutorSpec(intra_threads=threads))
    wall = time.perf_counter() - t0
    rec = _CFG["rec"][_CFG["k0"]]
    out = tl_record(res, _CFG["mi"], _CFG["li"], np.float64)
    np.savez_compressed(HERE / f"full_{name}.npz", frequency=f, mi=_CFG["mi"], li=_CFG["li"],
                        stride=cfg.options.output_stride, n_range=cfg.grid.n_range,
                        samples=np.stack(rec[0]), norms=np.array(rec[1]),
                        ref_seconds_per_step=wall / cfg.grid.n_range, ref_threads=threads, **out)
    print(f"{name}: {wall:.0f} s, {wall / cfg.grid.n_range:.3f} s/step (reference run_frequency)")


def farm(name, workers):
    """cfg4: all frequencies through the reference's own frequency_farm."""
    import tempfile
    cfg = configs.build(name)
    freqs = cfg.source.frequencies
    rec_dir = tempfile.mkdtemp(prefix="pe3d_full_")
    install(name, cfg, rec_dir)          # the forked workers inherit the rebinding
    t0 = time.perf_counter()
    report = pe3d.frequency_farm(ref_config(cfg, freqs), freqs, workers=workers, schedule="static")
    wall = time.perf_counter() - t0
    if report.failures:
        raise SystemExit(f"reference farm failures: {report.failures}")
    mi, li = _CFG["mi"], _CFG["li"]
    per = [tl_record(r, mi, li, np.float32) for r in report.results]
    samples, norms = [], []
    from paper_1711_00005_b200.environment import wavenumber
    for f in freqs:
        k0 = wavenumber(f, cfg.environment.c0)
        with np.load(Path(rec_dir) / f"rec_{k0!r}.npz") as z:
            samples.append(z["samples"])
            norms.append(z["norms"])
    stacked = {k: np.stack([p[k] for p in per]) for k in per[0]}
    np.savez_compressed(HERE / f"full_{name}.npz", frequencies=np.array(freqs), mi=mi, li=li,
                        stride=cfg.options.output_stride, n_range=cfg.grid.n_range,
                        samples=np.stack(samples), norms=np.stack(norms), workers=workers,
                        ref_wall_seconds=wall, **stacked)
    print(f"{name}: {len(freqs)} frequencies x {cfg.grid.n_range} steps in {wall:.0f} s "
          f"on {workers} reference workers")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=("cfg2", "cfg3", "cfg4", "cfg5"))
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--threads", type=int, default=1, help="reference intra_threads (single-frequency configs)")
    a = ap.parse_args()
    if a.config == "cfg4":
        farm(a.config, a.workers)
    else:
        single(a.config, a.threads)


if __name__ == "__main__":
    main()
