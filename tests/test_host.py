"""Host-side logic (no GPU): types, invariants, medium, configs, sharding
law, error mapping, stride/max_range rules."""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1711_00005_b200 import configs, errors
from paper_1711_00005_b200.config import ExecutorSpec, RunOptions
from paper_1711_00005_b200.environment import (
    PERIODIC, SECTOR, Absorber, Environment, Grid3D, SoundSpeedProfile, hankel_factor, is_range_independent,
    local_term_grid, refraction_index, transmission_loss_field, wavenumber,
)
from paper_1711_00005_b200.marching import default_output_stride, steps_within
from paper_1711_00005_b200.medium import ETA, Bathymetry, FluidBottom, LayeredMedium, Sponge
from paper_1711_00005_b200.operators import StepCoefficients
from paper_1711_00005_b200.parallel import block_ranges, rank_frequencies, static_assignment


def grid(**kw):
    args = dict(n_range=10, n_azimuth=8, n_depth=32, delta_r=5.0, delta_theta=2 * math.pi / 8,
                delta_z=4.0, r_start=5.0)
    args.update(kw)
    return Grid3D(**args)


class TestInvariants:
    @pytest.mark.parametrize("field", ["n_range", "n_azimuth", "n_depth"])
    def test_counts(self, field):
        with pytest.raises(errors.InvariantError, match=f"{field} >= 3"):
            grid(**{field: 2})

    def test_periodic_closure(self):
        with pytest.raises(errors.InvariantError, match="periodic closure"):
            grid(delta_theta=math.pi / 4, n_azimuth=4)

    def test_sector_no_closure(self):
        assert grid(azimuth_topology=SECTOR, delta_theta=math.radians(2)).azimuth_topology == SECTOR

    def test_coefficient_identities(self):
        c = StepCoefficients.for_step(wavenumber(50.0, 1500.0), 25.0)
        assert c.cx_lhs + c.cx_rhs == 0.5 + 0j and c.cy_lhs + c.cy_rhs == 0j
        with pytest.raises(errors.InvariantError):
            StepCoefficients(1j, 0.3, 0.3, 0, 0)

    def test_run_options(self):
        with pytest.raises(errors.InvariantError, match="output_stride"):
            RunOptions(output_stride=0)
        with pytest.raises(errors.InvariantError, match="intra_threads"):
            ExecutorSpec(intra_threads=0)


class TestGoldenScalars:
    """Reference golden values (ref tests/test_environment.py:66-258)."""

    def test_wavenumber(self):
        assert wavenumber(50.0, 1500.0) == pytest.approx(0.20943951023931956, rel=1e-14)

    def test_hankel_abs(self):
        assert abs(hankel_factor(0.3, 16.0)) == pytest.approx(0.25, rel=1e-14)

    def test_reference_refraction(self):
        g = grid()
        env = Environment(1500.0, SoundSpeedProfile.uniform(1600.0), 6000.0,
                          Absorber(0.75 * g.depth_extent, 0.01), g.depth_extent)
        n = refraction_index(env, 10.0, 0.0, g.depths())
        assert n.real[0] == pytest.approx(1500.0 / 1600.0, rel=1e-15)
        assert n.imag[-1] == pytest.approx(0.01, rel=1e-12) and n.imag[0] == 0.0

    def test_tl_floor(self):
        tl, clamped = transmission_loss_field(np.array([[0.0, 1.0]]), 1.0)
        assert tl[0, 0] == 300.0 and tl[0, 1] == 0.0 and clamped == 1


class TestMedium:
    def test_flat_medium_is_range_independent(self):
        for name in ("cfg1", "cfg2", "cfg4", "cfg5"):
            assert is_range_independent(configs.build(name, n_range=3).environment)
        assert not is_range_independent(configs.build("cfg3", n_range=3).environment)

    def test_attenuation_convention(self):
        g = grid(n_depth=64, delta_z=1.0)
        med = LayeredMedium(1500.0, SoundSpeedProfile.uniform(1500.0),
                            FluidBottom(1500.0, 1.0, 0.5, Bathymetry(1e9)))
        n = med.index_grid(g, 10.0, None)[0]
        assert n[0].imag == pytest.approx(0.0) and n[0].real == pytest.approx(1.0)
        deep = LayeredMedium(1500.0, SoundSpeedProfile.uniform(1500.0),
                             FluidBottom(1500.0, 1.0, 0.5, Bathymetry(-1e9)))
        assert deep.index_grid(g, 10.0, None)[0][40].imag == pytest.approx(ETA * 0.5, rel=1e-12)

    def test_density_needs_k0(self):
        cfg = configs.build("cfg1", n_range=3)
        with pytest.raises(errors.DomainError, match="k0"):
            local_term_grid(cfg.environment, cfg.grid, 5.0, None)
        loc = local_term_grid(cfg.environment, cfg.grid, 5.0, 0.2)
        assert loc.shape == (64, 256) and np.isfinite(loc).all()

    def test_sponge_ramp(self):
        g = grid(n_depth=64, delta_z=1.0)
        med = LayeredMedium(1500.0, SoundSpeedProfile.uniform(1500.0),
                            FluidBottom(1500.0, 1.0, 0.0, Bathymetry(1e9)), sponge=Sponge(8, 10.0))
        n = med.index_grid(g, 10.0, None)[0]
        assert np.all(n[:56].imag == 0) and np.all(np.diff(n[56:].imag) > 0)

    def test_configs_shapes(self):
        expect = {"cfg1": (64, 256, 1), "cfg2": (256, 2048, 1), "cfg3": (512, 512, 1),
                  "cfg4": (256, 1024, 64), "cfg5": (4096, 4096, 1)}
        for name, (nt, nz, nf) in expect.items():
            c = configs.build(name, n_range=3)
            assert (c.grid.n_azimuth, c.grid.n_depth, len(c.source.frequencies)) == (nt, nz, nf)

    def test_cfg4_frequencies_logspaced(self):
        f = configs.build("cfg4", n_range=3).source.frequencies
        assert f[0] == pytest.approx(50.0) and f[-1] == pytest.approx(500.0)
        assert np.allclose(np.diff(np.log(f)), math.log(10) / 63)


class TestMarchRules:
    def test_default_stride(self):
        assert [default_output_stride(n) for n in (10, 511, 512, 5000)] == [1, 1, 2, 10]

    def test_max_range_cut(self):
        g = grid(n_range=10, delta_r=5.0, r_start=5.0)
        assert steps_within(g, 26.0) == 4
        assert steps_within(g, None) == 10
        assert steps_within(g, 1.0) == 0


class TestStaticAssignment:
    def test_eight_three(self):
        assert static_assignment(8, 3) == [[0, 1, 2], [3, 4, 5], [6, 7]]

    def test_more_workers(self):
        assert [len(b) for b in static_assignment(2, 5)] == [1, 1, 0, 0, 0]

    @given(st.integers(0, 200), st.integers(1, 32))
    @settings(max_examples=200, deadline=None)
    def test_law(self, jobs, workers):
        blocks = static_assignment(jobs, workers)
        assert [i for b in blocks for i in b] == list(range(jobs))
        if jobs:
            assert max(len(b) for b in blocks) == math.ceil(jobs / workers)

    def test_block_ranges(self):
        assert block_ranges(8, 3) == [(0, 3), (3, 6), (6, 8)]

    def test_rank_frequencies_cover(self):
        freqs = list(range(64))
        for world in (1, 2, 4, 8, 3):
            got = [f for r in range(world) for f in rank_frequencies(freqs, r, world)]
            assert got == freqs


class TestErrorMapping:
    class Rec:
        def __init__(self, **kw):
            self.range_index, self.sweep, self.member, self.pivot, self.rank1 = -1, 0, 0, 0, 0
            self.message = b"boom\0"
            self.__dict__.update(kw)

    def test_singular_plain(self):
        with pytest.raises(errors.SingularSystemError) as info:
            errors.raise_from_record(1, self.Rec(member=7, pivot=3))
        assert info.value.member_index == 7 and info.value.pivot_index == 3

    def test_step_error(self):
        with pytest.raises(errors.StepError) as info:
            errors.raise_from_record(1, self.Rec(range_index=4, sweep=1, member=2))
        assert info.value.sweep == "azimuth" and info.value.range_index == 4
        assert isinstance(info.value.cause, errors.SingularSystemError)

    def test_cuda(self):
        with pytest.raises(errors.NativeError, match="boom"):
            errors.raise_from_record(3, self.Rec())

    def test_ok(self):
        errors.raise_from_record(0, self.Rec())


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4", "cfg5"])
def test_batched_host_columns_bitwise_equal_to_per_frequency(name):
    """The drop-in's host inputs for a batch of frequencies (starter columns and
    medium columns as one array expression each) equal, bit for bit, the
    per-frequency functions they replace (gaussian_starter_column, ref
    environment.py:270-284; the local term n^2 - 1 of the medium column)."""
    from paper_1711_00005_b200.environment import gaussian_starter_column, wavenumber
    from paper_1711_00005_b200.marching import _local_column, _local_columns, _starter_columns
    cfg = configs.build(name, n_range=5)
    grid, env, source, _ = cfg
    freqs = list(source.frequencies)[:7] + [f * 1.37 for f in source.frequencies[:2]]
    k0s = [wavenumber(f, env.c0) for f in freqs]
    got = _starter_columns(grid, source, k0s)
    want = np.stack([gaussian_starter_column(grid, source, k0) for k0 in k0s])
    assert got.tobytes() == want.tobytes()
    got = _local_columns(env, grid, grid.r_start, k0s)
    want = np.stack([_local_column(env, grid, grid.r_start, k0) for k0 in k0s])
    assert got.tobytes() == want.tobytes()
