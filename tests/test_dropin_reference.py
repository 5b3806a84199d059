"""The drop-in handed the REFERENCE's own objects on a GPU.

The unmodified reference package (baseline/_ref, the pip install of
/root/reference, which travels to the GPU box; see oracle/ref_harness.py)
builds ``pe3d.Config`` (ref config.py:98-102), ``pe3d.MarchState`` (ref
marching.py:48-62) and ``pe3d.SolveBatch`` (ref tridiag.py:82-142) objects;
the B200 ``run_frequency`` / ``range_step`` / ``frequency_farm`` /
``solve_batch`` take them unchanged, and their results are compared with
the reference's own functions run live on the same objects (cfg1-size grid,
the reference's own medium: sound-speed profile + quadratic absorber).
"""

import math

import numpy as np
import pytest

import paper_1711_00005_b200 as b200

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-9
TL_TOL = 1e-4


@pytest.fixture(scope="module")
def ref():
    from oracle import ref_harness
    try:
        return ref_harness.import_reference()
    except ImportError as exc:
        pytest.skip(f"reference not installed: {exc}")


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _tl(a, b):
    m = b < 150.0
    return float(np.abs(a - b)[m].max())


def _ref_config(ref, n_range=120, freqs=(50.0, 70.0), stride=10):
    grid = ref.Grid3D(n_range, 64, 256, 5.0, 2 * math.pi / 64, 1.0, 5.0)
    profile = ref.SoundSpeedProfile(np.array([0.0, 80.0, 256.0]), np.array([1500.0, 1490.0, 1530.0]))
    env = ref.Environment(1500.0, profile, 6000.0, ref.Absorber(0.8 * grid.depth_extent, 0.02),
                          grid.depth_extent)
    return ref.Config(grid, env, ref.SourceSpec(freqs, 50.0), ref.RunOptions(output_stride=stride))


def test_run_frequency_with_reference_config(ref):
    cfg = _ref_config(ref)
    want = ref.run_frequency(cfg, 70.0)
    got = b200.run_frequency(cfg, 70.0)
    assert np.array_equal(got.ranges, want.ranges) and got.output_stride == want.output_stride
    assert got.tl_field.shape == want.tl_field.shape
    assert _tl(got.tl_field, want.tl_field) <= TL_TOL
    assert _rel(got.final_slab.values, want.final_slab.values) <= FIELD_TOL
    assert got.final_slab.range_m == want.final_slab.range_m
    assert got.clamped_samples == want.clamped_samples


def test_range_step_with_reference_march_state(ref):
    cfg = _ref_config(ref, n_range=8)
    grid, env, src, _ = cfg
    k0 = ref.wavenumber(50.0, env.c0)
    coeffs = ref.StepCoefficients.for_step(k0, grid.delta_r)
    rng = np.random.default_rng(3)
    u0 = rng.standard_normal((64, 256)) + 1j * rng.standard_normal((64, 256))
    want = ref.MarchState(ref.FieldSlab(u0.copy(), grid.r_start), 0, coeffs, env, grid, k0)
    got = ref.MarchState(ref.FieldSlab(u0.copy(), grid.r_start), 0, coeffs, env, grid, k0)
    for _ in range(5):
        want = ref.range_step(want)
        got = b200.range_step(got)
        assert got.range_index == want.range_index and got.slab.range_m == want.slab.range_m
        assert _rel(got.slab.values, want.slab.values) <= FIELD_TOL


def test_frequency_farm_with_reference_config(ref):
    cfg = _ref_config(ref, n_range=60)
    want = ref.frequency_farm(cfg, [50.0, 70.0], workers=1)      # no fork from a CUDA process
    got = b200.frequency_farm(cfg, [50.0, 70.0], workers=2)
    assert got.ok and not want.failures
    for g, w in zip(got.results, want.results):
        assert g.frequency == w.frequency
        assert _tl(g.tl_field, w.tl_field) <= TL_TOL
        assert _rel(g.final_slab.values, w.final_slab.values) <= FIELD_TOL


def test_solve_batch_with_reference_batch(ref):
    from oracle import pe3d_oracle as O
    rng = np.random.default_rng(5)
    systems = [ref.TriDiagSystem(*O.random_system(rng, 40, True), ref.tridiag.CYCLIC) for _ in range(150)]
    batch = ref.SolveBatch.from_systems(systems)
    want = ref.solve_batch(batch, 4)
    got = b200.solve_batch(batch)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
