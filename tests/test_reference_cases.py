"""The reference's own unit cases for the hot path, restated against the
B200 package: same case names, same inputs by construction (seeded or by
hand), same expected behaviour.  Sources of the cases: ref
pkg/tests/test_tridiag.py (TestTriDiagSystem, TestSolveThomas,
TestSolveCyclic, TestSolveBatch, TestSolverProperties) and
pkg/tests/test_marching.py (TestApplyBoundary, TestRangeStep,
TestRunFrequency).  Cases already restated elsewhere are not repeated
(dense 3x3 step, lowest member across tiles, zero pivot, single unknown,
stride/max_range contract: tests/test_gpu_parity.py).

Host-only cases (type validation, apply_boundary) run without a GPU; the
rest call the CUDA kernels through the C ABI and are marked gpu.  Where the
reference compares its batch with its own scalar solver bit for bit, the
same invariant is asserted here on the GPU path (batch == scalar,
hint-invariant, member order free), and the values are compared with the
dense-elimination oracle at the reference's own 1e-10 criterion.
"""

import math

import numpy as np
import pytest

from oracle import pe3d_oracle as O
from paper_1711_00005_b200 import (
    Absorber, Environment, FieldSlab, Grid3D, MarchState, SoundSpeedProfile, SourceSpec, StepCoefficients,
    gaussian_starter, range_step, run_frequency, wavenumber,
)
from paper_1711_00005_b200.config import Config, RunOptions
from paper_1711_00005_b200.environment import PERIODIC, SECTOR
from paper_1711_00005_b200.errors import DomainError, InvariantError, ShapeError, SingularSystemError
from paper_1711_00005_b200.marching import apply_boundary
from paper_1711_00005_b200.tridiag import (
    CYCLIC, OPEN, SolveBatch, TriDiagSystem, solve_batch, solve_cyclic, solve_thomas,
)

gpu = pytest.mark.gpu


def rand_system(rng, n, topology):
    return TriDiagSystem(*O.random_system(rng, n, topology == CYCLIC), topology=topology)


def dense(system):
    return O.dense_solve(system.sub, system.main, system.sup, system.rhs, system.topology == CYCLIC)


def dense_matrix(s):
    n = s.n
    a = np.zeros((n, n), dtype=np.complex128)
    a[np.arange(n), np.arange(n)] = s.main
    if s.topology == CYCLIC:
        for i in range(n):
            a[i, (i - 1) % n] += s.sub[i]
            a[i, (i + 1) % n] += s.sup[i]
    else:
        a[np.arange(1, n), np.arange(n - 1)] = s.sub
        a[np.arange(n - 1), np.arange(1, n)] = s.sup
    return a


def make_grid(n_range=10, n_azimuth=8, n_depth=32, delta_r=5.0, delta_z=4.0, r_start=None, topology=PERIODIC):
    dth = 2 * math.pi / n_azimuth if topology == PERIODIC else math.radians(2.0)
    return Grid3D(n_range, n_azimuth, n_depth, delta_r, dth, delta_z, delta_r if r_start is None else r_start,
                  topology)


def make_env(grid, attenuation=0.01):
    return Environment(1500.0, SoundSpeedProfile.uniform(1500.0), 6000.0,
                       Absorber(0.75 * grid.depth_extent, attenuation), grid.depth_extent)


def make_config(options=None, source_depth=62.0, frequencies=(50.0,), **grid_kw):
    grid = make_grid(**grid_kw)
    return Config(grid, make_env(grid), SourceSpec(tuple(frequencies), source_depth), options or RunOptions())


def make_state(config, slab_values=None, delta_r=None, frequency=50.0):
    grid, env = config.grid, config.environment
    k0 = wavenumber(frequency, env.c0)
    coeffs = StepCoefficients.for_step(k0, grid.delta_r if delta_r is None else delta_r)
    slab = gaussian_starter(grid, config.source, k0) if slab_values is None else FieldSlab(slab_values, grid.r_start)
    return MarchState(slab, 0, coeffs, env, grid, k0)


def random_slab(rng, grid, zero_surface=True):
    v = rng.standard_normal((grid.n_azimuth, grid.n_depth)) + 1j * rng.standard_normal((grid.n_azimuth, grid.n_depth))
    if zero_surface:
        v[:, 0] = 0.0
    return v


# ------------------------------------------------ TestTriDiagSystem (host only)

class TestTriDiagSystem:
    def test_open_length_rules(self):
        with pytest.raises(ShapeError):
            TriDiagSystem(np.zeros(3), np.ones(3), np.zeros(2), np.ones(3), OPEN)

    def test_cyclic_length_rules(self):
        with pytest.raises(ShapeError):
            TriDiagSystem(np.zeros(2), np.ones(3), np.zeros(2), np.ones(3), CYCLIC)

    def test_cyclic_minimum_size(self):
        with pytest.raises(InvariantError, match="n >= 3"):
            TriDiagSystem(np.zeros(2), np.ones(2), np.zeros(2), np.ones(2), CYCLIC)

    def test_rhs_length(self):
        with pytest.raises(ShapeError):
            TriDiagSystem(np.zeros(2), np.ones(3), np.zeros(2), np.ones(4), OPEN)

    def test_empty_batch_rejected(self):
        with pytest.raises(InvariantError):
            SolveBatch.from_systems([])

    def test_mixed_sizes_rejected(self):
        rng = np.random.default_rng(7)
        with pytest.raises(InvariantError, match="share one n"):
            SolveBatch.from_systems([rand_system(rng, 5, OPEN), rand_system(rng, 6, OPEN)])

    def test_system_round_trip(self):
        rng = np.random.default_rng(8)
        systems = [rand_system(rng, 9, CYCLIC) for _ in range(4)]
        again = SolveBatch.from_systems(systems).system(2)
        assert np.array_equal(again.main, systems[2].main) and again.topology == CYCLIC

    def test_requires_matching_topology(self):
        # the topology check precedes any device work (ref tridiag.py:226, :240)
        rng = np.random.default_rng(0)
        with pytest.raises(DomainError):
            solve_thomas(rand_system(rng, 5, CYCLIC))
        with pytest.raises(DomainError):
            solve_cyclic(rand_system(rng, 5, OPEN))


# ---------------------------------------------------- TestApplyBoundary (host)

class TestApplyBoundary:
    def test_surface_row_zeroed(self):
        grid = make_grid()
        slab = FieldSlab(random_slab(np.random.default_rng(1), grid, zero_surface=False), grid.r_start)
        apply_boundary(slab, grid, make_env(grid))
        assert np.all(slab.values[:, 0] == 0.0)

    def test_periodic_leaves_azimuth_edges(self):
        grid = make_grid()
        values = random_slab(np.random.default_rng(2), grid, zero_surface=False)
        marker = values[0, 5]
        slab = FieldSlab(values, grid.r_start)
        apply_boundary(slab, grid, make_env(grid))
        assert slab.values[0, 5] == marker

    def test_sector_edges_zeroed(self):
        grid = make_grid(topology=SECTOR)
        slab = FieldSlab(random_slab(np.random.default_rng(3), grid, zero_surface=False), grid.r_start)
        apply_boundary(slab, grid, make_env(grid))
        assert np.all(slab.values[0, :] == 0.0) and np.all(slab.values[-1, :] == 0.0)

    def test_idempotent(self):
        grid = make_grid(topology=SECTOR)
        env = make_env(grid)
        slab = FieldSlab(random_slab(np.random.default_rng(4), grid, zero_surface=False), grid.r_start)
        once = apply_boundary(slab, grid, env).values.copy()
        assert np.array_equal(once, apply_boundary(slab, grid, env).values)


# ------------------------------------------------------ TestSolveThomas/Cyclic

@gpu
class TestSolveThomas:
    def test_identity_system(self):
        s = TriDiagSystem(np.zeros(2), np.ones(3), np.zeros(2), np.array([3.0, 4.0, 5.0]), OPEN)
        assert np.array_equal(solve_thomas(s), np.array([3.0, 4.0, 5.0]))

    def test_hand_solved_case(self):
        s = TriDiagSystem(np.array([-1.0, -1.0]), np.full(3, 2.0), np.array([-1.0, -1.0]),
                          np.array([1.0, 0.0, 1.0]), OPEN)
        x = solve_thomas(s)
        assert np.allclose(x, np.ones(3), rtol=1e-12)
        assert np.allclose(dense(s), x, rtol=1e-12)

    def test_random_against_oracle(self):
        s = rand_system(np.random.default_rng(101), 32, OPEN)
        ref = dense(s)
        assert np.max(np.abs(solve_thomas(s) - ref)) <= 1e-10 * np.max(np.abs(ref))


@gpu
class TestSolveCyclic:
    def test_row_sum_case(self):
        s = TriDiagSystem(np.full(3, -1.0), np.full(3, 3.0), np.full(3, -1.0), np.ones(3), CYCLIC)
        x = solve_cyclic(s)
        assert np.allclose(x, np.ones(3), rtol=1e-12)
        assert np.allclose(dense(s), x, rtol=1e-12)

    def test_zero_corners_degenerate_to_open(self):
        o = rand_system(np.random.default_rng(7), 16, OPEN)
        cyc = TriDiagSystem(np.concatenate([[0.0], o.sub]), o.main.copy(), np.concatenate([o.sup, [0.0]]),
                            o.rhs.copy(), CYCLIC)
        assert np.allclose(solve_cyclic(cyc), solve_thomas(o), rtol=1e-12)

    def test_random_against_oracle(self):
        s = rand_system(np.random.default_rng(202), 32, CYCLIC)
        ref = dense(s)
        assert np.max(np.abs(solve_cyclic(s) - ref)) <= 1e-10 * np.max(np.abs(ref))


# ------------------------------------------------------------- TestSolveBatch

@gpu
class TestSolveBatch:
    def test_batch_of_one_equals_scalar(self):
        s = rand_system(np.random.default_rng(1), 32, OPEN)
        assert solve_batch(SolveBatch.from_systems([s]))[0].tobytes() == solve_thomas(s).tobytes()

    def test_identical_members_identical_solutions(self):
        s = rand_system(np.random.default_rng(2), 24, OPEN)
        x = solve_batch(SolveBatch.from_systems([s] * 100))
        assert np.array_equal(x, np.broadcast_to(x[0], x.shape))

    def test_hint_invariance_and_scalar_agreement(self):
        rng = np.random.default_rng(3)
        systems = [rand_system(rng, 40, OPEN) for _ in range(900)]
        batch = SolveBatch.from_systems(systems)
        base = solve_batch(batch, parallel_hint=1)
        for hint in (2, 8):
            assert base.tobytes() == solve_batch(batch, parallel_hint=hint).tobytes()
        # a member's bits do not depend on its position or its neighbours
        for i in (0, 63, 64, 511, 899):
            assert base[i].tobytes() == solve_thomas(systems[i]).tobytes()
        ref = O.solve_batch(batch.sub, batch.main, batch.sup, batch.rhs, cyclic=False)
        assert np.max(np.abs(base - ref)) <= 1e-12 * np.max(np.abs(ref))

    def test_cyclic_batch_matches_scalar(self):
        rng = np.random.default_rng(4)
        systems = [rand_system(rng, 17, CYCLIC) for _ in range(130)]
        batch = SolveBatch.from_systems(systems)
        x = solve_batch(batch, parallel_hint=3)
        for i in (0, 1, 64, 65, 129):
            assert x[i].tobytes() == solve_cyclic(systems[i]).tobytes()
        ref = O.solve_batch(batch.sub, batch.main, batch.sup, batch.rhs, cyclic=True)
        assert np.max(np.abs(x - ref)) <= 1e-12 * np.max(np.abs(ref))

    def test_singular_member_named_no_partial_result(self):
        rng = np.random.default_rng(5)
        systems = [rand_system(rng, 8, OPEN) for _ in range(10)]
        systems[7] = TriDiagSystem(np.ones(7), np.zeros(8), np.ones(7), np.ones(8), OPEN)
        with pytest.raises(SingularSystemError) as info:
            solve_batch(SolveBatch.from_systems(systems))
        assert info.value.member_index == 7

    def test_bad_hint_rejected(self):
        s = rand_system(np.random.default_rng(9), 8, OPEN)
        with pytest.raises(InvariantError):
            solve_batch(SolveBatch.from_systems([s]), parallel_hint=0)


@gpu
class TestSolverProperties:
    def test_residual_bound_random_instances(self):
        rng = np.random.default_rng(404)
        for _ in range(150):
            n = int(rng.integers(3, 129))
            topology = OPEN if rng.random() < 0.5 else CYCLIC
            s = rand_system(rng, n, topology)
            x = solve_thomas(s) if topology == OPEN else solve_cyclic(s)
            bound = 1e-10 * max(1.0, np.max(np.abs(s.rhs)))
            assert np.max(np.abs(dense_matrix(s) @ x - s.rhs)) <= bound

    def test_linearity_in_rhs(self):
        rng = np.random.default_rng(505)
        base = rand_system(rng, 48, OPEN)
        r1 = rng.standard_normal(48) + 1j * rng.standard_normal(48)
        r2 = rng.standard_normal(48) + 1j * rng.standard_normal(48)
        a, b = 0.7 - 1.1j, -2.0 + 0.4j

        def solve(rhs):
            return solve_thomas(TriDiagSystem(base.sub.copy(), base.main.copy(), base.sup.copy(), rhs, OPEN))

        x1, x2, x12 = solve(r1), solve(r2), solve(a * r1 + b * r2)
        assert np.max(np.abs(x12 - (a * x1 + b * x2))) <= 1e-10 * np.max(np.abs(x12))


# --------------------------------------------------------------- TestRangeStep

@gpu
class TestRangeStep:
    def test_delta_zero_identity_bitwise(self):
        config = make_config(n_azimuth=8, n_depth=24)
        values = random_slab(np.random.default_rng(5), config.grid)
        state = make_state(config, slab_values=values.copy(), delta_r=0.0)
        before = state.slab.values.copy()
        after = range_step(state)
        assert after.range_index == 1
        assert after.slab.values.tobytes() == before.tobytes()

    def test_advances_range_and_index(self):
        config = make_config(n_azimuth=6, n_depth=24)
        new = range_step(make_state(config))
        assert new.range_index == 1 and new.slab.range_m == config.grid.range_at(1)

    def test_azimuth_symmetry_preserved_one_step(self):
        config = make_config(n_azimuth=16, n_depth=48)
        mags = np.abs(range_step(make_state(config)).slab.values)
        assert (mags.max(axis=0) - mags.min(axis=0)).max() <= 1e-12 * mags.max()

    def test_surface_zero_after_step(self):
        out = range_step(make_state(make_config()))
        assert np.all(out.slab.values[:, 0] == 0.0)

    def test_state_range_invariant(self):
        config = make_config(n_range=4)
        state = make_state(config)
        for j in range(1, 5):
            state = range_step(state)
            assert state.slab.range_m == config.grid.range_at(j) and state.range_index == j

    def test_input_state_untouched(self):
        # range_step returns a new state; the caller's slab is not modified (ref marching.py:93-136)
        config = make_config(n_azimuth=8, n_depth=24)
        state = make_state(config)
        before = state.slab.values.copy()
        range_step(state)
        assert state.slab.values.tobytes() == before.tobytes() and state.range_index == 0


# ------------------------------------------------------------ TestRunFrequency

@gpu
class TestRunFrequency:
    def test_rerun_bitwise_identical(self):
        config = make_config(n_range=6, n_azimuth=8, n_depth=32)
        first, second = run_frequency(config, 50.0), run_frequency(config, 50.0)
        assert first.tl_field.tobytes() == second.tl_field.tobytes()
        assert first.final_slab.values.tobytes() == second.final_slab.values.tobytes()
        assert np.array_equal(first.ranges, second.ranges)

    def test_no_blowup_with_absorber(self):
        config = make_config(n_range=100, n_azimuth=8, n_depth=64, delta_z=4.0, source_depth=100.0)
        starter_max = math.sqrt(wavenumber(50.0, config.environment.c0))
        result = run_frequency(config, 50.0)
        assert np.max(np.abs(result.final_slab.values)) <= 10.0 * starter_max

    def test_tl_field_finite(self):
        assert np.all(np.isfinite(run_frequency(make_config(n_range=5), 50.0).tl_field))

    def test_run_equals_repeated_range_step(self):
        # run_frequency is range_step applied n_range times to the starter (ref marching.py:176-183)
        config = make_config(n_range=5, n_azimuth=8, n_depth=32, options=RunOptions(output_stride=1))
        state = make_state(config)
        for _ in range(5):
            state = range_step(state)
        res = run_frequency(config, 50.0)
        err = np.linalg.norm(res.final_slab.values - state.slab.values) / np.linalg.norm(state.slab.values)
        assert err <= 1e-12
        assert res.final_slab.range_m == state.slab.range_m
