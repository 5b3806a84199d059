"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every fixture records outputs of the unmodified reference ``pe3d``
(``/root/reference/pkg/src``).  For the BASELINE media, which the
reference cannot express, the reference's march is driven with the
shared medium of ``paper_1711_00005_b200.medium`` injected by rebinding
``pe3d.marching.refraction_index_grid`` (ref ``marching.py:31,110,116``);
everything else -- operators, assembly, Thomas/Sherman-Morrison solves,
boundary handling, TL -- is the reference's own code.

The fixtures are small (sparse samples + norms at full grid sizes) so
they travel with the repo; the GPU tests compare against them without
needing the reference on the GPU box.
"""

from __future__ import annotations

import math
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import pe3d                                      # noqa: E402  (the reference)
import pe3d.errors                               # noqa: E402
import pe3d.marching as ref_marching             # noqa: E402
from pe3d.selftest import random_system          # noqa: E402

from paper_1711_00005_b200 import configs        # noqa: E402
from paper_1711_00005_b200.environment import refraction_index_grid, wavenumber  # noqa: E402

SAMPLE_POINTS = 1024


def ref_grid(g):
    return pe3d.Grid3D(g.n_range, g.n_azimuth, g.n_depth, g.delta_r, g.delta_theta,
                       g.delta_z, g.r_start, g.azimuth_topology)


def ref_env(grid, c0=1500.0):
    return pe3d.Environment(c0, pe3d.SoundSpeedProfile.uniform(c0), 6000.0,
                            pe3d.Absorber(0.0, 0.0), grid.depth_extent)


def inject(env, grid, k0):
    """Rebind the reference's n-grid lookup to the shared medium."""
    ref_marching.refraction_index_grid = lambda e, g, r: refraction_index_grid(env, grid, r, k0)


def restore():
    ref_marching.refraction_index_grid = pe3d.environment.refraction_index_grid


def tridiag_fixture():
    rng = np.random.default_rng(1001)
    out = {}
    for tag, topo, count in (("open", pe3d.tridiag.OPEN, 40), ("cyclic", pe3d.tridiag.CYCLIC, 40)):
        ns, subs, mains, sups, rhss, xs, dense = [], [], [], [], [], [], []
        for _ in range(count):
            n = int(rng.integers(3, 129))
            s = random_system(rng, n, topo)
            x = pe3d.solve_thomas(s) if topo == pe3d.tridiag.OPEN else pe3d.solve_cyclic(s)
            ns.append(n)
            subs.append(s.sub); mains.append(s.main); sups.append(s.sup); rhss.append(s.rhs)
            xs.append(x); dense.append(pe3d.dense_oracle_solve(s))
        out[f"{tag}_n"] = np.array(ns)
        for key, arrs in (("sub", subs), ("main", mains), ("sup", sups), ("rhs", rhss),
                          ("x", xs), ("dense", dense)):
            out[f"{tag}_{key}"] = np.concatenate(arrs)
    # one batch through solve_batch (shared n, 130 members, 3 threads)
    systems = [random_system(rng, 17, pe3d.tridiag.CYCLIC) for _ in range(130)]
    batch = pe3d.SolveBatch.from_systems(systems)
    out["batch_sub"], out["batch_main"] = batch.sub, batch.main
    out["batch_sup"], out["batch_rhs"] = batch.sup, batch.rhs
    out["batch_x"] = pe3d.solve_batch(batch, parallel_hint=3)
    np.savez_compressed(HERE / "tridiag_systems.npz", **out)


def dense_step_fixture():
    """Criterion 2 inputs/outputs (ref tests/test_acceptance.py:72-116)."""
    rng = np.random.default_rng(1002)
    grid = pe3d.Grid3D(10, 3, 3, 4.0, 2 * math.pi / 3, 7.0, 30.0)
    env = pe3d.Environment(1500.0, pe3d.SoundSpeedProfile.uniform(1500.0), 6000.0,
                           pe3d.Absorber(0.5 * grid.depth_extent, 0.0), grid.depth_extent)
    k0 = pe3d.wavenumber(50.0, 1500.0)
    coeffs = pe3d.StepCoefficients.for_step(k0, grid.delta_r)
    u0 = rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3))
    u0[:, 0] = 0.0
    state = pe3d.MarchState(pe3d.FieldSlab(u0.copy(), grid.r_start), 0, coeffs, env, grid, k0)
    out = pe3d.range_step(state).slab.values
    np.savez_compressed(HERE / "dense_step_3x3.npz", u0=u0, out=out, k0=k0)


def small_march_fixture(topology):
    """Reference medium (profile + quadratic absorber), random start slab,
    30 steps, every slab recorded -- periodic and sector grids."""
    rng = np.random.default_rng(7 if topology == "periodic" else 8)
    n_az, n_dep = 8, 32
    dth = 2 * math.pi / n_az if topology == "periodic" else math.radians(2.0)
    grid = pe3d.Grid3D(30, n_az, n_dep, 5.0, dth, 4.0, 5.0, topology)
    profile = pe3d.SoundSpeedProfile(np.array([0.0, 60.0, 124.0]), np.array([1500.0, 1490.0, 1520.0]))
    env = pe3d.Environment(1500.0, profile, 6000.0,
                           pe3d.Absorber(0.75 * grid.depth_extent, 0.01), grid.depth_extent)
    k0 = pe3d.wavenumber(50.0, 1500.0)
    coeffs = pe3d.StepCoefficients.for_step(k0, grid.delta_r)
    u0 = rng.standard_normal((n_az, n_dep)) + 1j * rng.standard_normal((n_az, n_dep))
    state = pe3d.MarchState(pe3d.FieldSlab(u0.copy(), grid.r_start), 0, coeffs, env, grid, k0)
    slabs = []
    for _ in range(grid.n_range):
        state = pe3d.range_step(state)
        slabs.append(state.slab.values.copy())
    np.savez_compressed(HERE / f"small_march_{topology}.npz", u0=u0, slabs=np.stack(slabs),
                        k0=k0, profile_z=profile.depths, profile_c=profile.speeds)


def cfg1_full_fixture():
    """cfg1 at full length through the reference's run_frequency."""
    cfg = configs.build("cfg1")
    g, env = cfg.grid, cfg.environment
    k0 = wavenumber(50.0, env.c0)
    inject(env, g, k0)
    try:
        rcfg = pe3d.Config(ref_grid(g), ref_env(g), pe3d.SourceSpec((50.0,), cfg.source.depth),
                           pe3d.RunOptions(output_stride=cfg.options.output_stride))
        res = pe3d.run_frequency(rcfg, 50.0)
    finally:
        restore()
    tl = res.tl_field
    np.savez_compressed(HERE / "cfg1_full.npz", ranges=res.ranges, tl_theta0=tl[:, 0, :],
                        tl_theta_spread=np.ptp(tl, axis=1).max(),
                        clamped=res.clamped_samples, final=res.final_slab.values)


def full_size_fixture(name, frequency, n_steps):
    """A few steps at the config's full grid size, every step sampled at
    SAMPLE_POINTS seeded points plus per-step norms and theta-0 column."""
    cfg = configs.build(name, n_range=n_steps, frequencies=(frequency,))
    g, env = cfg.grid, cfg.environment
    k0 = wavenumber(frequency, env.c0)
    rng = np.random.default_rng(4242)
    mi = rng.integers(0, g.n_azimuth, SAMPLE_POINTS)
    li = rng.integers(0, g.n_depth, SAMPLE_POINTS)
    inject(env, g, k0)
    try:
        rg = ref_grid(g)
        src = pe3d.SourceSpec((frequency,), cfg.source.depth)
        slab = pe3d.gaussian_starter(rg, src, k0)
        state = pe3d.MarchState(slab, 0, pe3d.StepCoefficients.for_step(k0, g.delta_r),
                                ref_env(g), rg, k0)
        samples, norms, col0, sums = [], [], [], []
        t0 = time.perf_counter()
        for _ in range(n_steps):
            state = pe3d.range_step(state)
            u = state.slab.values
            samples.append(u[mi, li])
            norms.append(np.linalg.norm(u))
            sums.append(u.sum())
        wall = time.perf_counter() - t0
    finally:
        restore()
    np.savez_compressed(HERE / f"{name}_f{int(frequency)}_{n_steps}steps.npz",
                        frequency=frequency, mi=mi, li=li, samples=np.stack(samples),
                        norms=np.array(norms), sums=np.array(sums), col0=state.slab.values[0].copy(),
                        ref_seconds_per_step=wall / n_steps)
    print(f"{name} f={frequency}: {wall / n_steps:.2f} s/step (reference)")


def azimuth_singular_fixture():
    """Hand-built step coefficients whose periodic azimuth system is singular
    for the reference's Sherman-Morrison solve (diag = 0: StepError at the
    azimuth sweep, pivot n - 1) or degenerate without tripping its checks
    (diag = 2 off: no error) -- ref marching.py:124-131, tridiag.py:145-212."""
    grid = pe3d.Grid3D(10, 8, 16, 5.0, 2 * math.pi / 8, 4.0, 5.0)
    env = pe3d.Environment(1500.0, pe3d.SoundSpeedProfile.uniform(1500.0), 6000.0,
                           pe3d.Absorber(0.75 * grid.depth_extent, 0.01), grid.depth_extent)
    k0 = 0.2
    s = 1.0 / ((k0 * grid.range_at(1)) * grid.delta_theta) ** 2
    base = pe3d.StepCoefficients.for_step(k0, grid.delta_r)
    out = {"k0": k0, "cx_lhs": base.cx_lhs, "cx_rhs": base.cx_rhs, "delta": base.delta}
    for tag, c in (("diag0", 1 / (2 * s)), ("diag2off", 1 / (4 * s))):
        co = pe3d.StepCoefficients(delta=base.delta, cx_lhs=base.cx_lhs, cx_rhs=base.cx_rhs, cy_lhs=complex(c),
                                   cy_rhs=-complex(c))
        state = pe3d.MarchState(pe3d.FieldSlab(np.ones((8, 16), complex), grid.r_start), 0, co, env, grid, k0)
        out[f"{tag}_cy"] = complex(c)
        try:
            with np.errstate(all="ignore"):
                pe3d.range_step(state)
            out[f"{tag}_error"] = np.array([0, -1, -1, -1])
        except pe3d.errors.StepError as e:
            cause = e.__cause__
            out[f"{tag}_error"] = np.array([1, e.range_index, e.member_index, cause.pivot_index])
            assert e.sweep == "azimuth"
    np.savez_compressed(HERE / "azimuth_singular.npz", **out)


def output_fixture():
    """TL files written by the reference's own writers (ref output.py:60-122)
    for a fixed small result, plus the inputs that produced them."""
    import math as _m
    import pe3d.output as ref_out
    out = HERE / "output"
    out.mkdir(exist_ok=True)
    grid = pe3d.Grid3D(10, 4, 5, 5.0, 2 * _m.pi / 4, 3.0, 5.0)
    rng = np.random.default_rng(77)
    tl = 40.0 + 30.0 * rng.random((3, 4, 5))
    tl[1, 2, 3] = 300.0
    final = rng.standard_normal((4, 5)) + 1j * rng.standard_normal((4, 5))
    res = pe3d.FrequencyResult(frequency=63.5, ranges=np.array([5.0, 15.0, 25.0]), tl_field=tl, clamped_samples=1,
                               final_slab=pe3d.FieldSlab(final, 25.0), output_stride=2, wall_seconds=0.5)
    ref_out.write_tl_csv(out / "ref_tl.csv", res, grid)
    ref_out.write_tl_binary(out / "ref_tl.bin", res, grid)
    ref_out.write_manifest(out, {"command": "run", "frequencies": [{"frequency_hz": 63.5, "sha256": "x"}],
                                 "grid": {"n_range": 10}})
    np.savez_compressed(out / "inputs.npz", tl=tl, ranges=res.ranges)


def main(which=None):
    jobs = {
        "tridiag": tridiag_fixture,
        "dense": dense_step_fixture,
        "small": lambda: (small_march_fixture("periodic"), small_march_fixture("sector")),
        "cfg1": cfg1_full_fixture,
        "output": output_fixture,
        "azsing": azimuth_singular_fixture,
        "cfg2": lambda: full_size_fixture("cfg2", 100.0, 20),
        "cfg3": lambda: full_size_fixture("cfg3", 25.0, 20),
        "cfg4": lambda: (full_size_fixture("cfg4", 50.0, 10), full_size_fixture("cfg4", 500.0, 10)),
        "cfg5": lambda: full_size_fixture("cfg5", 500.0, 3),
    }
    for key, fn in jobs.items():
        if which and key not in which:
            continue
        t = time.perf_counter()
        fn()
        print(f"{key}: {time.perf_counter() - t:.1f} s")


if __name__ == "__main__":
    main(sys.argv[1:])
