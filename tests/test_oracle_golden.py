"""Pin the CPU oracle (oracle/pe3d_oracle.py) to outputs of the reference
package itself (fixtures written by tests/golden/make_golden.py)."""

import math

import numpy as np
import pytest

from oracle import pe3d_oracle as O
from paper_1711_00005_b200 import configs
from paper_1711_00005_b200.environment import (
    PERIODIC, SECTOR, Absorber, Environment, Grid3D, SoundSpeedProfile, local_term_grid, wavenumber,
)


def _systems(fx, tag):
    ns = fx[f"{tag}_n"]
    off = 0
    offo = 0
    for n in ns:
        n = int(n)
        n_off = n if tag == "cyclic" else n - 1
        yield (fx[f"{tag}_sub"][offo:offo + n_off], fx[f"{tag}_main"][off:off + n],
               fx[f"{tag}_sup"][offo:offo + n_off], fx[f"{tag}_rhs"][off:off + n],
               fx[f"{tag}_x"][off:off + n], fx[f"{tag}_dense"][off:off + n])
        off += n
        offo += n_off


@pytest.mark.parametrize("tag", ["open", "cyclic"])
def test_tridiag_systems_match_reference(golden, tag):
    fx = golden("tridiag_systems.npz")
    for sub, main, sup, rhs, x_ref, dense_ref in _systems(fx, tag):
        cyc = tag == "cyclic"
        x = O.solve_batch(sub[:, None], main[:, None], sup[:, None], rhs[:, None], cyclic=cyc)[0]
        assert np.array_equal(x, x_ref) or np.abs(x - x_ref).max() <= 1e-15 * np.abs(x_ref).max()
        d = O.dense_solve(sub, main, sup, rhs, cyclic=cyc)
        assert np.abs(d - dense_ref).max() <= 1e-13 * np.abs(dense_ref).max()
        assert np.abs(x - d).max() <= 1e-10 * np.abs(d).max()   # criterion 1 bound


def test_batch_fixture(golden):
    fx = golden("tridiag_systems.npz")
    x = O.solve_batch(fx["batch_sub"], fx["batch_main"], fx["batch_sup"], fx["batch_rhs"], cyclic=True)
    assert np.abs(x - fx["batch_x"]).max() <= 1e-15 * np.abs(fx["batch_x"]).max()


def test_singular_lowest_member():
    rng = np.random.default_rng(6)
    systems = [O.random_system(rng, 6, False) for _ in range(200)]
    bad = (np.ones(5), np.zeros(6), np.ones(5), np.ones(6))
    systems[70] = systems[150] = bad
    arrs = [np.stack([s[k] for s in systems], axis=1) for k in range(4)]
    with pytest.raises(O.OracleSingular) as info:
        O.solve_batch(*arrs, cyclic=False)
    assert info.value.member == 70 and info.value.pivot == 0


def test_dense_step_3x3(golden):
    fx = golden("dense_step_3x3.npz")
    geo = O.StepGeometry(3, 3, 2 * math.pi / 3, 7.0, True)
    k0 = float(fx["k0"])
    d = 1j * (k0 * 4.0)
    q = d / 4.0
    out, _ = O.range_step(fx["u0"].copy(), 0, 30.0, 34.0, k0, (d, 0.25 - q, 0.25 + q, -q, q),
                          0.0, 0.0, geo)
    assert np.abs(out - fx["out"]).max() <= 1e-15 * np.abs(fx["out"]).max()


@pytest.mark.parametrize("topology", [PERIODIC, SECTOR])
def test_small_march(golden, topology):
    fx = golden(f"small_march_{topology}.npz")
    n_az, n_dep = 8, 32
    dth = 2 * math.pi / n_az if topology == PERIODIC else math.radians(2.0)
    grid = Grid3D(30, n_az, n_dep, 5.0, dth, 4.0, 5.0, topology)
    env = Environment(1500.0, SoundSpeedProfile(fx["profile_z"], fx["profile_c"]), 6000.0,
                      Absorber(0.75 * grid.depth_extent, 0.01), grid.depth_extent)
    k0 = float(fx["k0"])
    local = local_term_grid(env, grid, grid.r_start, k0)
    geo = O.StepGeometry(n_az, n_dep, dth, 4.0, topology == PERIODIC)
    d = 1j * (k0 * 5.0)
    q = d / 4.0
    u, r = fx["u0"].copy(), grid.r_start
    for j in range(30):
        u, r = O.range_step(u, j, r, grid.range_at(j + 1), k0, (d, 0.25 - q, 0.25 + q, -q, q),
                            local, local, geo)
        ref = fx["slabs"][j]
        assert np.abs(u - ref).max() <= 1e-14 * np.abs(ref).max(), f"step {j + 1}"


def test_cfg1_full_length(golden):
    fx = golden("cfg1_full.npz")
    cfg = configs.build("cfg1")
    res = O.run_frequency(cfg, 50.0)
    assert np.array_equal(res.ranges, fx["ranges"])
    assert res.clamped == int(fx["clamped"])
    err = np.linalg.norm(res.final - fx["final"]) / np.linalg.norm(fx["final"])
    assert err <= 1e-13
    assert np.abs(res.tl_field[:, 0, :] - fx["tl_theta0"]).max() <= 1e-9


FIXTURE_STEPS = {"cfg2": 20, "cfg3": 20, "cfg4": 10, "cfg5": 3}


@pytest.mark.parametrize("name,freq,steps", [("cfg2", 100.0, 20), ("cfg4", 50.0, 10),
                                             ("cfg4", 500.0, 10), ("cfg3", 25.0, 6),
                                             ("cfg5", 500.0, 1)])
def test_full_size_steps(golden, name, freq, steps):
    fx = golden(f"{name}_f{int(freq)}_{FIXTURE_STEPS[name]}steps.npz")
    cfg = configs.build(name, n_range=max(steps, 3), frequencies=(freq,))
    g, env = cfg.grid, cfg.environment
    k0 = wavenumber(freq, env.c0)
    geo = O.StepGeometry(g.n_azimuth, g.n_depth, g.delta_theta, g.delta_z, True)
    d = 1j * (k0 * g.delta_r)
    q = d / 4.0
    from paper_1711_00005_b200.environment import gaussian_starter
    u = gaussian_starter(g, cfg.source, k0).values.copy()
    r = g.r_start
    for j in range(steps):
        rn = g.range_at(j + 1)
        u, r = O.range_step(u, j, r, rn, k0, (d, 0.25 - q, 0.25 + q, -q, q),
                            local_term_grid(env, g, r, k0), local_term_grid(env, g, rn, k0), geo)
        s = fx["samples"][j]
        got = u[fx["mi"], fx["li"]]
        assert np.linalg.norm(got - s) <= 1e-13 * np.linalg.norm(s)
        assert abs(np.linalg.norm(u) - fx["norms"][j]) <= 1e-13 * fx["norms"][j]
