"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden fixtures and the CPU oracle.

Contract (BASELINE.json north_star): field relative L2 <= 1e-9 and
|dTL| <= 1e-4 dB wherever TL < 150 dB, at every output range.  Tighter
bounds are used where the reference's own tests pin them (criteria 1, 2,
4 of ref tests/test_acceptance.py).
"""

import math

import numpy as np
import pytest

from oracle import pe3d_oracle as O
from paper_1711_00005_b200 import (
    Absorber, Environment, FieldSlab, Grid3D, MarchState, SoundSpeedProfile, SourceSpec, StepCoefficients,
    configs, gaussian_starter, march_frequencies, range_step, run_frequency, wavenumber,
)
from paper_1711_00005_b200 import _native
from paper_1711_00005_b200.config import Config, RunOptions
from paper_1711_00005_b200.environment import PERIODIC, SECTOR
from paper_1711_00005_b200.errors import DomainError, SingularSystemError, StepError
from paper_1711_00005_b200.tridiag import CYCLIC, OPEN, SolveBatch, TriDiagSystem, solve_batch, solve_cyclic, solve_thomas

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-9
TL_TOL = 1e-4


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def tl_err(a, b):
    mask = b < 150.0
    return float(np.abs(a - b)[mask].max()) if mask.any() else 0.0


def make_grid(n_range=10, n_azimuth=8, n_depth=32, delta_r=5.0, delta_z=4.0, r_start=None, topology=PERIODIC):
    dth = 2 * math.pi / n_azimuth if topology == PERIODIC else math.radians(2.0)
    return Grid3D(n_range, n_azimuth, n_depth, delta_r, dth, delta_z, delta_r if r_start is None else r_start,
                  topology)


def make_env(grid, attenuation=0.01, start_frac=0.75, profile=None):
    return Environment(1500.0, profile or SoundSpeedProfile.uniform(1500.0), 6000.0,
                       Absorber(start_frac * grid.depth_extent, attenuation), grid.depth_extent)


# ------------------------------------------------------------ solve_batch

def _fixture_systems(fx, tag):
    off = offo = 0
    for n in fx[f"{tag}_n"]:
        n = int(n)
        n_off = n if tag == "cyclic" else n - 1
        yield TriDiagSystem(fx[f"{tag}_sub"][offo:offo + n_off], fx[f"{tag}_main"][off:off + n],
                            fx[f"{tag}_sup"][offo:offo + n_off], fx[f"{tag}_rhs"][off:off + n],
                            OPEN if tag == "open" else CYCLIC), fx[f"{tag}_x"][off:off + n]
        off += n
        offo += n_off


@pytest.mark.parametrize("tag", ["open", "cyclic"])
def test_solve_matches_reference_solutions(golden, tag):
    fx = golden("tridiag_systems.npz")
    for system, x_ref in _fixture_systems(fx, tag):
        x = solve_thomas(system) if tag == "open" else solve_cyclic(system)
        assert np.abs(x - x_ref).max() <= 1e-12 * np.abs(x_ref).max()


def test_criterion_01_random_systems_vs_dense():
    rng = np.random.default_rng(1001)
    for cyclic in (False, True):
        for _ in range(100):
            n = int(rng.integers(3, 129))
            sub, main, sup, rhs = O.random_system(rng, n, cyclic)
            x = solve_batch(SolveBatch(sub[:, None], main[:, None], sup[:, None], rhs[:, None],
                                       CYCLIC if cyclic else OPEN))[0]
            ref = O.dense_solve(sub, main, sup, rhs, cyclic)
            assert np.abs(x - ref).max() <= 1e-10 * np.abs(ref).max()


def test_batch_fixture_broadcast_and_order(golden):
    fx = golden("tridiag_systems.npz")
    x = solve_batch(SolveBatch(fx["batch_sub"], fx["batch_main"], fx["batch_sup"], fx["batch_rhs"], CYCLIC))
    assert np.abs(x - fx["batch_x"]).max() <= 1e-12 * np.abs(fx["batch_x"]).max()
    # broadcast views (stride 0), as assemble_azimuth_batch builds them
    n, w = 17, 40
    rng = np.random.default_rng(3)
    rhs = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    b = SolveBatch(np.broadcast_to(np.complex128(0.3 - 0.1j), (n, w)),
                   np.broadcast_to(np.complex128(2.0 + 1j), (n, w)),
                   np.broadcast_to(np.complex128(0.3 - 0.1j), (n, w)), rhs, CYCLIC)
    x = solve_batch(b)
    ref = O.solve_batch(b.sub, b.main, b.sup, b.rhs, cyclic=True)
    assert np.abs(x - ref).max() <= 1e-13 * np.abs(ref).max()


def test_singular_lowest_member_across_tiles():
    rng = np.random.default_rng(6)
    systems = [TriDiagSystem(*O.random_system(rng, 6, False)) for _ in range(200)]
    bad = TriDiagSystem(np.ones(5), np.zeros(6), np.ones(5), np.ones(6))
    systems[70] = systems[150] = bad
    with pytest.raises(SingularSystemError) as info:
        solve_batch(SolveBatch.from_systems(systems), parallel_hint=4)
    assert info.value.member_index == 70 and info.value.pivot_index == 0


def test_zero_pivot_and_single_unknown():
    with pytest.raises(SingularSystemError) as info:
        solve_thomas(TriDiagSystem(np.ones(2), np.zeros(3), np.ones(2), np.ones(3)))
    assert info.value.pivot_index == 0
    assert solve_thomas(TriDiagSystem(np.zeros(0), np.array([2.0]), np.zeros(0), np.array([5.0])))[0] == 2.5
    x = solve_cyclic(TriDiagSystem(np.full(3, -1.0), np.full(3, 3.0), np.full(3, -1.0), np.ones(3), CYCLIC))
    assert np.allclose(x, 1.0, rtol=1e-12)


# ------------------------------------------------------------ range_step

def test_criterion_02_dense_step_3x3(golden):
    fx = golden("dense_step_3x3.npz")
    grid = Grid3D(10, 3, 3, 4.0, 2 * math.pi / 3, 7.0, 30.0)
    env = make_env(grid, attenuation=0.0, start_frac=0.5)
    k0 = float(fx["k0"])
    state = MarchState(FieldSlab(fx["u0"].copy(), 30.0), 0, StepCoefficients.for_step(k0, 4.0), env, grid, k0)
    out = range_step(state).slab.values
    assert np.abs(out - fx["out"]).max() <= 1e-12 * np.abs(fx["out"]).max()


def test_criterion_03_delta_zero_bitwise():
    rng = np.random.default_rng(1003)
    grid = make_grid()
    env = make_env(grid)
    v = rng.standard_normal((8, 32)) + 1j * rng.standard_normal((8, 32))
    v[:, 0] = 0
    k0 = wavenumber(50.0, 1500.0)
    state = MarchState(FieldSlab(v.copy(), grid.r_start), 0, StepCoefficients.for_step(k0, 0.0), env, grid, k0)
    after = range_step(state)
    assert after.range_index == 1 and after.slab.values.tobytes() == v.tobytes()


@pytest.mark.parametrize("topology", [PERIODIC, SECTOR])
def test_small_march_every_step(golden, topology):
    fx = golden(f"small_march_{topology}.npz")
    grid = make_grid(n_range=30, n_azimuth=8, n_depth=32, delta_r=5.0, delta_z=4.0, r_start=5.0, topology=topology)
    env = make_env(grid, profile=SoundSpeedProfile(fx["profile_z"], fx["profile_c"]))
    k0 = float(fx["k0"])
    state = MarchState(FieldSlab(fx["u0"].copy(), grid.r_start), 0, StepCoefficients.for_step(k0, 5.0),
                       env, grid, k0)
    for j in range(30):
        state = range_step(state)
        assert rel_l2(state.slab.values, fx["slabs"][j]) <= 1e-12, f"step {j + 1}"
        assert state.slab.range_m == grid.range_at(j + 1)


@pytest.mark.parametrize("topology", [PERIODIC, SECTOR])
@pytest.mark.parametrize("n_azimuth,n_depth", [(3, 3), (5, 7), (33, 9), (100, 13), (96, 1023), (600, 61)])
def test_ragged_grids_vs_oracle(topology, n_azimuth, n_depth):
    """Grids that are not multiples of the tile (8 rows), the warp (32) or the
    ring chunk sizes, down to the 3 x 3 minimum, through the march kernels
    (pad rows, partial ring chunks, block/direct ring paths) against the
    oracle at every output range."""
    grid = make_grid(n_range=6, n_azimuth=n_azimuth, n_depth=n_depth, delta_r=5.0, delta_z=2.0, r_start=5.0,
                     topology=topology)
    env = make_env(grid)
    src = SourceSpec((50.0, 90.0), 0.4 * grid.depth_extent)
    cfg = Config(grid, env, src, RunOptions(output_stride=2))
    got = march_frequencies(cfg, [50.0, 90.0])
    for r in got:
        ref = O.run_frequency(cfg, r.frequency)
        assert rel_l2(r.final_slab.values, ref.final) <= FIELD_TOL
        assert tl_err(r.tl_field, ref.tl_field) <= TL_TOL
        assert r.tl_field.shape == ref.tl_field.shape


@pytest.mark.parametrize("n_azimuth,n_depth", [(768, 40), (1280, 24), (4000, 16), (64, 1500), (32, 2050), (96, 4096)])
def test_ragged_wide_and_deep_grids_vs_oracle(n_azimuth, n_depth):
    """The wide-ring (clusters of 3 and 5 segments, the direct kernel at
    4000 azimuths) and long-column paths (1500 and 2050 rows: the 512-thread
    TMA column kernel; 4096 rows: the cluster column kernel) on ragged sizes,
    against the oracle."""
    grid = make_grid(n_range=3, n_azimuth=n_azimuth, n_depth=n_depth, delta_r=5.0, delta_z=1.0, r_start=5.0)
    env = make_env(grid)
    cfg = Config(grid, env, SourceSpec((60.0,), 0.4 * grid.depth_extent), RunOptions(output_stride=1))
    r = march_frequencies(cfg, [60.0])[0]
    ref = O.run_frequency(cfg, 60.0)
    assert rel_l2(r.final_slab.values, ref.final) <= FIELD_TOL
    assert tl_err(r.tl_field, ref.tl_field) <= TL_TOL


def test_singular_depth_becomes_step_error():
    grid = make_grid(n_azimuth=4, n_depth=8, delta_z=1.0)
    env = make_env(grid)
    coeffs = StepCoefficients(delta=1j, cx_lhs=0.5 + 0j, cx_rhs=0j, cy_lhs=0j, cy_rhs=0j)
    state = MarchState(FieldSlab(np.ones((4, 8), dtype=complex), grid.r_start), 0, coeffs, env, grid, 1.0)
    with pytest.raises(StepError) as info:
        range_step(state)
    assert info.value.sweep == "depth" and info.value.range_index == 1 and info.value.member_index == 0


def test_step_beyond_grid_rejected():
    grid = make_grid(n_range=3)
    env = make_env(grid)
    k0 = wavenumber(50.0, 1500.0)
    state = MarchState(gaussian_starter(grid, SourceSpec((50.0,), 60.0), k0), 0,
                       StepCoefficients.for_step(k0, grid.delta_r), env, grid, k0)
    for _ in range(3):
        state = range_step(state)
    with pytest.raises(DomainError, match="n_range"):
        range_step(state)


# ------------------------------------------------------------ run_frequency

def test_cfg1_full_length_vs_reference(golden):
    fx = golden("cfg1_full.npz")
    res = run_frequency(configs.build("cfg1"), 50.0)
    assert np.array_equal(res.ranges, fx["ranges"])
    assert rel_l2(res.final_slab.values, fx["final"]) <= FIELD_TOL
    assert tl_err(res.tl_field[:, 0, :], fx["tl_theta0"]) <= TL_TOL
    # azimuth independent medium + starter: every azimuth carries the same TL
    assert np.ptp(res.tl_field, axis=1).max() <= 1e-6


def test_snapshots_every_output_range_vs_oracle():
    cfg = configs.build("cfg1", n_range=60, frequencies=(50.0, 65.0), output_stride=10)
    for r in march_frequencies(cfg, [50.0, 65.0], keep_snapshots=True):
        ref = O.run_frequency(cfg, r.frequency, keep_snapshots=True)
        assert r.snapshots.shape == ref.snapshots.shape
        for s in range(ref.snapshots.shape[0]):
            assert rel_l2(r.snapshots[s], ref.snapshots[s]) <= FIELD_TOL, s
        assert tl_err(r.tl_field, ref.tl_field) <= TL_TOL
        assert r.clamped_samples == ref.clamped


FULL = {"cfg2": (100.0, 20), "cfg4a": (50.0, 10), "cfg4b": (500.0, 10), "cfg5": (500.0, 3), "cfg3": (25.0, 20)}


@pytest.mark.parametrize("key", ["cfg2", "cfg4a", "cfg4b", "cfg5", "cfg3"])
def test_full_size_steps_vs_reference(golden, key):
    name = key[:4]
    freq, steps = FULL[key]
    fx = golden(f"{name}_f{int(freq)}_{steps}steps.npz")
    cfg = configs.build(name, n_range=steps, frequencies=(freq,), output_stride=1)
    r = march_frequencies(cfg, [freq], keep_snapshots=True)[0]
    for j in range(steps):
        u = r.snapshots[j + 1]
        got = u[fx["mi"], fx["li"]]
        assert np.linalg.norm(got - fx["samples"][j]) <= FIELD_TOL * np.linalg.norm(fx["samples"][j]), j
        assert abs(np.linalg.norm(u) - fx["norms"][j]) <= FIELD_TOL * fx["norms"][j]
    assert rel_l2(r.final_slab.values[0], fx["col0"]) <= FIELD_TOL


def test_serial_and_scan_paths_agree():
    cfg = configs.build("cfg4", n_range=12, frequencies=(50.0, 200.0), output_stride=4)
    a = march_frequencies(cfg, [50.0, 200.0])
    b = march_frequencies(cfg, [50.0, 200.0], flags=_native.FLAG_SERIAL)
    for x, y in zip(a, b):
        assert rel_l2(x.final_slab.values, y.final_slab.values) <= 1e-11
        assert tl_err(x.tl_field, y.tl_field) <= 1e-8


def test_batch_equals_single_and_rerun_bitwise():
    cfg = configs.build("cfg4", n_range=8, frequencies=(50.0, 90.0, 300.0), output_stride=4)
    batch = march_frequencies(cfg, [50.0, 90.0, 300.0])
    single = march_frequencies(cfg, [90.0])[0]
    again = march_frequencies(cfg, [50.0, 90.0, 300.0])
    assert batch[1].final_slab.values.tobytes() == single.final_slab.values.tobytes()
    assert batch[1].tl_field.tobytes() == single.tl_field.tobytes()
    for x, y in zip(batch, again):
        assert x.final_slab.values.tobytes() == y.final_slab.values.tobytes()


@pytest.mark.parametrize("n_azimuth,chunk", [(768, None), (1024, None), (2048, None), (4096, None), (4096, "8")])
def test_cluster_ring_matches_direct_ring(monkeypatch, n_azimuth, chunk):
    """Wide rings: the thread-block-cluster azimuth sweep (segments of 512 or
    256 azimuths joined over DSMEM, cluster sizes 2..16) against the one-CTA
    direct kernel (PE3D_RING_BLOCK) on the same march, and both against the
    oracle on a short run."""
    cfg = configs.build("cfg5", n_range=4, output_stride=2)
    grid = cfg.grid
    small = Config(Grid3D(4, n_azimuth, 128, grid.delta_r, 2 * math.pi / n_azimuth, grid.delta_z, grid.r_start),
                   cfg.environment, SourceSpec((500.0,), 30.0), RunOptions(output_stride=2))
    monkeypatch.delenv("PE3D_RING_BLOCK", raising=False)
    if chunk:
        monkeypatch.setenv("PE3D_CLUSTER_L", chunk)
    got = march_frequencies(small, [500.0], flags=_native.FLAG_NO_GRAPH)[0]
    monkeypatch.setenv("PE3D_RING_BLOCK", "1")
    ref = march_frequencies(small, [500.0], flags=_native.FLAG_NO_GRAPH)[0]
    # different (both exact) summation orders; near r = 0 the rings are
    # ill-conditioned (rho -> 1), so allow rounding growth well inside 1e-9
    assert rel_l2(got.final_slab.values, ref.final_slab.values) <= 1e-10
    assert tl_err(got.tl_field, ref.tl_field) <= 1e-8
    if n_azimuth == 1024:
        orc = O.run_frequency(small, 500.0)
        assert rel_l2(got.final_slab.values, orc.final) <= 1e-9
        assert tl_err(got.tl_field, orc.tl_field) <= 1e-4


@pytest.mark.parametrize("n_depth,topology", [(2048, PERIODIC), (4096, PERIODIC), (4096, SECTOR)])
def test_cluster_depth_sweep_matches_single_cta(monkeypatch, n_depth, topology):
    """Long columns: the depth sweep split over a cluster of 1024-row
    sub-columns (carries over DSMEM, halo rows from global) against the
    one-CTA-per-column kernel, and against the oracle."""
    cfg = configs.build("cfg5", n_range=4, output_stride=2)
    grid = cfg.grid
    small = Config(Grid3D(4, 64, n_depth, grid.delta_r, 2 * math.pi / 64, grid.delta_z, grid.r_start,
                          azimuth_topology=topology),
                   cfg.environment, SourceSpec((500.0,), 600.0), RunOptions(output_stride=2))
    monkeypatch.delenv("PE3D_DEPTH_NO_CLUSTER", raising=False)
    got = march_frequencies(small, [500.0], flags=_native.FLAG_NO_GRAPH)[0]
    monkeypatch.setenv("PE3D_DEPTH_NO_CLUSTER", "1")
    ref = march_frequencies(small, [500.0], flags=_native.FLAG_NO_GRAPH)[0]
    assert rel_l2(got.final_slab.values, ref.final_slab.values) <= 1e-12
    assert tl_err(got.tl_field, ref.tl_field) <= 1e-9
    orc = O.run_frequency(small, 500.0)
    assert rel_l2(got.final_slab.values, orc.final) <= FIELD_TOL
    assert tl_err(got.tl_field, orc.tl_field) <= TL_TOL


@pytest.mark.parametrize("family", ["split_cluster", "split_halo", "lockstep_cluster", "warp_chains"])
def test_async_kernels_race_stress(monkeypatch, family):
    """Race stress for the asynchronous kernels (compute-sanitizer is closed on
    this GPU pool, profiles/r02_compute_sanitizer_closed.txt): TMA producer /
    consumer mbarrier rings, DSMEM st.async exchanges, the split-column
    carries.  Twenty marches per family, graphed and unGraphed, must be
    bitwise identical -- the split sweeps with the corrected cluster ring
    (cfg5 shape), the same from 400 m on, where every step runs the halo-form
    split-ring kernel (segment + neighbour granules on one mbarrier), the
    lock-step cluster sweeps, and the ring-per-warp TMA sweep with 1, 2 and 8
    concurrent step chains (cfg4 shape)."""
    if family == "warp_chains":
        cfg = configs.build("cfg4", n_range=6, frequencies=(50.0, 80.0, 130.0, 200.0, 310.0, 420.0, 460.0, 500.0),
                            output_stride=3)
        freqs = list(cfg.source.frequencies)
        settings = [(c, fl) for c in ("1", "2", "8") for fl in (0, _native.FLAG_NO_GRAPH)] * 4
    else:
        if family == "lockstep_cluster":
            monkeypatch.setenv("PE3D_DEPTH_NO_SPLIT", "1")
        cfg5 = configs.build("cfg5", n_range=6, output_stride=3)
        grid = cfg5.grid
        r_start = 400.0 if family == "split_halo" else grid.r_start
        cfg = Config(Grid3D(6, 2048, 4096, grid.delta_r, 2 * math.pi / 2048, grid.delta_z, r_start),
                     cfg5.environment, SourceSpec((500.0,), 600.0), RunOptions(output_stride=3))
        freqs = [500.0]
        settings = [(None, fl) for fl in (0, _native.FLAG_NO_GRAPH)] * 10
    first = None
    for chains, flags in settings:
        if chains:
            monkeypatch.setenv("PE3D_CHAINS", chains)
        runs = march_frequencies(cfg, freqs, flags=flags)
        got = [(r.final_slab.values.tobytes(), r.tl_field.tobytes(), r.clamped_samples) for r in runs]
        if first is None:
            first = got
        assert got == first


@pytest.mark.parametrize("nranks", [2, 4])
def test_cluster_ring_slab_layout(nranks):
    """The cluster kernel on rank-chunked depth slabs (virtual ranks) equals
    the undecomposed march with the same kernel."""
    from paper_1711_00005_b200 import slab_march
    cfg = configs.build("cfg5", n_range=4, output_stride=2)
    grid = cfg.grid
    small = Config(Grid3D(4, 2048, 256, grid.delta_r, 2 * math.pi / 2048, grid.delta_z, grid.r_start),
                   cfg.environment, SourceSpec((500.0,), 30.0), RunOptions(output_stride=2))
    ref = march_frequencies(small, [500.0])[0]
    got = slab_march(small, 500.0, nranks)
    assert got.final.tobytes() == ref.final_slab.values.tobytes()
    assert got.tl_field.tobytes() == ref.tl_field.tobytes()


@pytest.mark.parametrize("chains", ["2", "3", "8"])
def test_concurrent_chains_bitwise_equal_to_one_chain(monkeypatch, chains):
    """Disjoint frequency groups marched as concurrent graph branches
    (PE3D_CHAINS) give bitwise the single-chain results: TL at every output
    range, clamped counts and final slabs, with uneven groups (5 = 2+3 or
    1+2+2 frequencies) and one chain per frequency (8, clamped to 5)."""
    freqs = (50.0, 90.0, 150.0, 300.0, 500.0)
    cfg = configs.build("cfg4", n_range=8, frequencies=freqs, output_stride=2)
    monkeypatch.setenv("PE3D_CHAINS", "1")
    ref = march_frequencies(cfg, list(freqs))
    monkeypatch.setenv("PE3D_CHAINS", chains)
    got = march_frequencies(cfg, list(freqs))
    for x, y in zip(ref, got):
        assert x.tl_field.tobytes() == y.tl_field.tobytes()
        assert x.final_slab.values.tobytes() == y.final_slab.values.tobytes()
        assert x.clamped_samples == y.clamped_samples


@pytest.mark.parametrize("n_steps,stride", [(2, 5), (6, 3), (9, 4)])
def test_march_graph_variants_bitwise_equal(monkeypatch, n_steps, stride):
    """The march's round-2 launch forms against their plain counterparts, bitwise:
    the final slab stored by TMA from the azimuth sweep's stage (reference layout,
    PE3D_FINAL_STORES: per-element stores), the parameters carried by one kernel
    node (PE3D_PARAMS_MEMCPY: copies from page-locked staging), the write-only
    prologue of a column starter (PE3D_PREPARE_STAGED: the staged prologue) and the
    first depth sweep reading the starter's temp column (PE3D_FIRST_STEP_FIELD: the
    azimuth-uniform temp field).  Final step with and without a TL sample; two chains."""
    freqs = (50.0, 170.0, 420.0)
    cfg = configs.build("cfg4", n_range=max(n_steps, 3), frequencies=freqs, output_stride=stride)

    def run():
        res = march_frequencies(cfg, list(freqs), n_steps=n_steps)
        return [(r.tl_field.tobytes(), r.final_slab.values.tobytes(), r.clamped_samples) for r in res]

    monkeypatch.setenv("PE3D_CHAINS", "2")
    ref = None
    switches = ("PE3D_FINAL_STORES", "PE3D_PARAMS_MEMCPY", "PE3D_PREPARE_STAGED", "PE3D_FIRST_STEP_FIELD")
    for switch in (None,) + switches:
        for name in switches:
            monkeypatch.delenv(name, raising=False)
        if switch:
            monkeypatch.setenv(switch, "1")
        got = run()
        if ref is None:
            ref = got
        else:
            assert got == ref, switch


@pytest.mark.parametrize("n_theta,n_depth,r_start", [(1024, 1024, 400.0), (2048, 2048, 400.0), (4096, 1024, 400.0),
                                                     (4096, 2048, 190.0), (1024, 512, 700.0)])
def test_split_rings_match_cluster_sweep(monkeypatch, n_theta, n_depth, r_start):
    """Split-ring steps (every 512-point ring segment solved on all SMs, its carries
    taken from the neighbouring segments' points loaded with it, TL steps included)
    against the cluster kernel on every step: the cfg5 medium where the carries only
    reach the segment edges (spans of 86-20 points: three, two and one halo
    granules), 2 to 8 segments, with and without split depth columns, TL every 4
    steps."""
    import dataclasses
    cfg = configs.build("cfg5", n_range=12, output_stride=4)
    grid, env, source, options = cfg
    grid = dataclasses.replace(grid, n_azimuth=n_theta, n_depth=n_depth, delta_theta=2 * math.pi / n_theta,
                               r_start=r_start)
    cfg = Config(grid, env, dataclasses.replace(source, depth=min(source.depth, 0.4 * grid.depth_extent)), options)
    f = cfg.source.frequencies[0]
    monkeypatch.setenv("PE3D_NO_SPLIT_RING", "1")
    ref = march_frequencies(cfg, [f])[0]
    monkeypatch.delenv("PE3D_NO_SPLIT_RING")
    got = march_frequencies(cfg, [f])[0]
    assert rel_l2(got.final_slab.values, ref.final_slab.values) <= 1e-12
    assert tl_err(got.tl_field, ref.tl_field) <= 1e-9
    assert got.clamped_samples == ref.clamped_samples


@pytest.mark.parametrize("groups,n_freq", [("2", 7), ("3", 7), ("4", 7), ("3", 12)])
def test_grouped_host_march_bitwise_equal(monkeypatch, groups, n_freq):
    """pe3d_march_host marching its frequencies in groups (each group's final slab
    copied out while the next marches; PE3D_HOST_GROUPS) against one march of all
    of them: bitwise equal TL, final slabs and clamped counts, with uneven groups
    (7 and 12 frequencies) and TL streamed to page-locked memory; each group's final
    slab is queued behind its last kernel, before the host waits for the march."""
    freqs = (50.0, 80.0, 130.0, 170.0, 260.0, 340.0, 500.0, 65.0, 95.0, 210.0, 300.0, 420.0)[:n_freq]
    cfg = configs.build("cfg4", n_range=6, frequencies=freqs, output_stride=2)

    def run():
        res = march_frequencies(cfg, list(freqs))
        return [(r.tl_field.tobytes(), r.final_slab.values.tobytes(), r.clamped_samples) for r in res]

    monkeypatch.setenv("PE3D_HOST_GROUPS", "1")
    ref = run()
    monkeypatch.setenv("PE3D_HOST_GROUPS", groups)
    assert run() == ref
    # grouped marches of column starters send only the first azimuth row of the
    # starting TL sample and replicate it on the host (pe3d_abi.cu RowReplicator):
    # the same bytes as the full copy (PE3D_TL0_FULL), whatever the thread count
    import ctypes as C

    def d2h_bytes():
        b_in, b_out = C.c_int64(0), C.c_int64(0)
        _native.load_library().pe3d_last_copy_bytes(_native.handle(0), C.byref(b_in), C.byref(b_out))
        assert b_in.value == len(freqs) * 2 * 1024 * 16          # starter and medium columns
        return b_out.value

    slab, S = 256 * 1024, 4
    full = len(freqs) * (S * slab * 8 + slab * 16 + 8)
    monkeypatch.setenv("PE3D_TL0_THREADS", "3")
    assert run() == ref
    assert d2h_bytes() == (full - len(freqs) * (slab - 1024) * 8 if int(groups) > 1 else full)
    monkeypatch.delenv("PE3D_TL0_THREADS")
    monkeypatch.setenv("PE3D_TL0_FULL", "1")
    assert run() == ref
    assert d2h_bytes() == full


@pytest.mark.parametrize("shape", ["cfg4", "long"])
def test_depth_setup_table_bitwise_equal_to_in_kernel_setup(monkeypatch, shape):
    """The per-march depth-sweep setup records (k_depth_setup /
    k_depth_setup_cluster, bulk-copied at a frequency switch) against the
    in-kernel frequency setup (PE3D_NO_K1_TABLE): bitwise equal TL, final
    slabs and clamped counts, several frequencies per CTA (switches), for
    1024-row columns (k_depth_tma) and 2048-row columns (the cluster sweep)."""
    freqs = (50.0, 90.0, 150.0)
    if shape == "cfg4":
        cfg = configs.build("cfg4", n_range=6, frequencies=freqs, output_stride=3)
    else:
        grid = make_grid(n_range=6, n_azimuth=512, n_depth=2048, delta_r=2.0, delta_z=0.5, r_start=2.0)
        cfg = Config(grid, make_env(grid), SourceSpec(freqs, 0.3 * grid.depth_extent), RunOptions(output_stride=3))
    if shape == "long":
        monkeypatch.setenv("PE3D_DEPTH_NO_SPLIT", "1")     # the cluster sweep (the split sweep needs the table)
    monkeypatch.setenv("PE3D_NO_K1_TABLE", "1")
    ref = march_frequencies(cfg, list(freqs))
    monkeypatch.delenv("PE3D_NO_K1_TABLE")
    got = march_frequencies(cfg, list(freqs))
    for x, y in zip(ref, got):
        assert x.tl_field.tobytes() == y.tl_field.tobytes()
        assert x.final_slab.values.tobytes() == y.final_slab.values.tobytes()
        assert x.clamped_samples == y.clamped_samples


@pytest.mark.parametrize("n_depth,n_azimuth", [(2048, 256), (4096, 512), (3072, 1024)])
def test_split_columns_match_cluster_sweep_and_oracle(monkeypatch, n_depth, n_azimuth):
    """Long columns solved as independent 1024-row sub-columns with exact
    carries applied by the azimuth sweep (LaunchCtx::split, the default for
    cfg2/cfg5 shapes) against the lock-step cluster sweep
    (PE3D_DEPTH_NO_SPLIT) and the CPU oracle: several frequencies (chains and
    frequency switches), TL at every output range."""
    freqs = (40.0, 75.0)
    grid = make_grid(n_range=8, n_azimuth=n_azimuth, n_depth=n_depth, delta_r=2.0, delta_z=0.5, r_start=2.0)
    cfg = Config(grid, make_env(grid), SourceSpec(freqs, 0.3 * grid.depth_extent), RunOptions(output_stride=2))
    got = march_frequencies(cfg, list(freqs), keep_snapshots=True)
    monkeypatch.setenv("PE3D_DEPTH_NO_SPLIT", "1")
    ref = march_frequencies(cfg, list(freqs), keep_snapshots=True)
    for x, y in zip(got, ref):
        assert rel_l2(x.final_slab.values, y.final_slab.values) <= 1e-12
        assert tl_err(x.tl_field, y.tl_field) <= 1e-9
        assert x.clamped_samples == y.clamped_samples
    o = O.run_frequency(cfg, freqs[1], keep_snapshots=True)
    assert rel_l2(got[1].final_slab.values, o.final) <= FIELD_TOL
    assert tl_err(got[1].tl_field, o.tl_field) <= TL_TOL


@pytest.mark.parametrize("shape", ["cfg4", "cfg2"])
def test_programmatic_launch_bitwise_equal(monkeypatch, shape):
    """The step sweeps launched with programmatic dependent launch (default)
    against plain stream-ordered launches (PE3D_NO_PDL): bitwise equal TL,
    final slabs and clamped counts -- the 1024-row column sweep with eight
    chains (8 frequencies) and the 2048-row cluster sweep (cfg2)."""
    if shape == "cfg4":
        freqs = (50.0, 70.0, 90.0, 120.0, 150.0, 200.0, 300.0, 500.0)
        cfg = configs.build("cfg4", n_range=8, frequencies=freqs, output_stride=4)
    else:
        freqs = (100.0,)
        cfg = configs.build("cfg2", n_range=8, output_stride=4)
    got = march_frequencies(cfg, list(freqs))
    monkeypatch.setenv("PE3D_NO_PDL", "1")
    ref = march_frequencies(cfg, list(freqs))
    for x, y in zip(ref, got):
        assert x.tl_field.tobytes() == y.tl_field.tobytes()
        assert x.final_slab.values.tobytes() == y.final_slab.values.tobytes()
        assert x.clamped_samples == y.clamped_samples


@pytest.mark.parametrize("name,freq,n_steps", [("cfg4", 500.0, 300), ("cfg2", 100.0, 150), ("cfg3", 25.0, 150)])
def test_full_size_long_march_vs_oracle(name, freq, n_steps):
    """BASELINE grids at full size over longer marches than the golden
    fixtures (cfg4's highest frequency for 300 steps, cfg2 and cfg3 for 150),
    against the oracle run here: the contract (field relative L2 <= 1e-9,
    |dTL| <= 1e-4 dB where TL < 150 dB) at every output range, i.e. the
    rounding drift of the scan formulations stays inside it."""
    if name == "cfg4":
        cfg = configs.build(name, n_range=n_steps, frequencies=(freq,), output_stride=50)
    else:
        cfg = configs.build(name, n_range=n_steps, output_stride=50)
    got = march_frequencies(cfg, [freq], keep_snapshots=True)[0]
    ref = O.run_frequency(cfg, freq, keep_snapshots=True)
    assert got.tl_field.shape == ref.tl_field.shape
    for k in range(ref.tl_field.shape[0]):
        assert rel_l2(got.snapshots[k], ref.snapshots[k]) <= FIELD_TOL, f"sample {k}"
        assert tl_err(got.tl_field[k], ref.tl_field[k]) <= TL_TOL, f"sample {k}"
    assert rel_l2(got.final_slab.values, ref.final) <= FIELD_TOL


def test_parallel_factorization_matches_reference_recurrence(monkeypatch):
    """The depth tables from the continuant scan (one CTA per frequency)
    against the reference-order single-thread Thomas recurrence."""
    cfg = configs.build("cfg4", n_range=10, frequencies=(50.0, 120.0, 500.0), output_stride=5)
    monkeypatch.setenv("PE3D_FACTOR_SERIAL", "1")
    ref = march_frequencies(cfg, [50.0, 120.0, 500.0], flags=_native.FLAG_NO_GRAPH)
    monkeypatch.delenv("PE3D_FACTOR_SERIAL")
    got = march_frequencies(cfg, [50.0, 120.0, 500.0], flags=_native.FLAG_NO_GRAPH)
    for x, y in zip(ref, got):
        assert rel_l2(y.final_slab.values, x.final_slab.values) <= 1e-12
        assert tl_err(y.tl_field, x.tl_field) <= 1e-9


@pytest.mark.parametrize("n_steps,stride,chains,topology", [
    (0, 1, "2", PERIODIC), (5, 10, "2", PERIODIC), (5, 10, "1", PERIODIC), (6, 6, "2", PERIODIC),
    (6, 2, "1", PERIODIC), (21, 3, "2", PERIODIC),
    (21, 3, "3", PERIODIC), (21, 3, "8", PERIODIC), (13, 2, "1", SECTOR)])
def test_tl_streaming_to_pinned_host(monkeypatch, n_steps, stride, chains, topology):
    """pe3d_march_host with a page-locked TL stack streams the samples through
    a device ring (R = min(S, 4) slots, copies overlapping the march, ring
    wrap-around when S > 4; a graphed loop that records no sample, S = 1):
    bitwise the stack copied after the march."""
    import ctypes as C
    import torch
    from paper_1711_00005_b200.marching import _grid_params, _local_column
    from paper_1711_00005_b200.environment import gaussian_starter
    monkeypatch.setenv("PE3D_CHAINS", chains)
    freqs = (50.0, 90.0, 150.0, 300.0)
    grid = make_grid(n_range=max(n_steps, 3), n_azimuth=64, n_depth=96, delta_r=5.0, delta_z=2.0, r_start=5.0,
                     topology=topology)
    env = make_env(grid)
    src = SourceSpec(freqs, 0.4 * grid.depth_extent)
    k0s = [wavenumber(f, 1500.0) for f in freqs]
    coeffs = _native.make_coeffs(k0s, [StepCoefficients.for_step(k0, grid.delta_r) for k0 in k0s])
    local = np.ascontiguousarray(np.stack([_local_column(env, grid, grid.r_start, k0) for k0 in k0s]))
    u0 = np.ascontiguousarray(np.stack([gaussian_starter(grid, src, k0).values for k0 in k0s]))
    S = 1 + n_steps // stride
    F, NT, NZ = len(freqs), grid.n_azimuth, grid.n_depth

    def run(streamed):
        if streamed:
            monkeypatch.delenv("PE3D_NO_TL_STREAM", raising=False)
        else:
            monkeypatch.setenv("PE3D_NO_TL_STREAM", "1")
        tl = torch.empty((F, S, NT, NZ), dtype=torch.float64).pin_memory()
        fin = torch.empty((F, NT, NZ * 2), dtype=torch.float64).pin_memory()
        cl = torch.zeros(F, dtype=torch.int64).pin_memory()
        g = _grid_params(grid, F, n_steps, stride, 0, grid.r_start)
        _native.call("pe3d_march_host", _native.handle(), g, coeffs, _native.ptr(local), _native.ptr(u0),
                     C.c_void_p(fin.data_ptr()), C.c_void_p(tl.data_ptr()), None, C.c_void_p(cl.data_ptr()))
        return tl.numpy().copy(), fin.numpy().copy(), cl.numpy().copy()

    a, b = run(True), run(False)
    for x, y in zip(a, b):
        assert x.tobytes() == y.tobytes()
    assert np.isfinite(a[0]).all()


def test_run_frequency_contract():
    grid = make_grid(n_range=10, delta_r=5.0, r_start=5.0)
    env = make_env(grid)
    src = SourceSpec((50.0,), 62.0)
    res = run_frequency(Config(grid, env, src, RunOptions(output_stride=4)), 50.0)
    assert res.tl_field.shape == (3, 8, 32) and res.output_stride == 4
    res = run_frequency(Config(grid, env, src, RunOptions(max_range=26.0, output_stride=1)), 50.0)
    assert res.final_slab.range_m == 25.0 and res.tl_field.shape[0] == 5
    res = run_frequency(Config(grid, env, src, RunOptions(max_range=1.0, output_stride=1)), 50.0)
    assert res.ranges.tolist() == [5.0] and res.tl_field.shape[0] == 1
    with pytest.raises(DomainError, match="not one of the source"):
        run_frequency(Config(grid, env, src, RunOptions()), 60.0)
    assert np.all(np.isfinite(res.tl_field))


def test_criterion_04_azimuth_symmetry_100_steps():
    grid = make_grid(n_range=100, n_azimuth=64, n_depth=256, delta_r=5.0, delta_z=4.0, r_start=5.0)
    env = make_env(grid)
    cfg = Config(grid, env, SourceSpec((50.0,), 200.0), RunOptions(output_stride=1))
    r = march_frequencies(cfg, [50.0], keep_snapshots=True)[0]
    for s in r.snapshots[1:]:
        mags = np.abs(s)
        assert (mags.max(axis=0) - mags.min(axis=0)).max() <= 1e-9 * mags.max()


def test_criterion_05_cylindrical_spreading():
    grid = Grid3D(3200, 8, 65, 5.0, 2 * math.pi / 8, 3.125, 5.0)
    env = Environment(1500.0, SoundSpeedProfile.uniform(1500.0), 6000.0, Absorber(0.9 * grid.depth_extent, 0.0),
                      grid.depth_extent)
    res = run_frequency(Config(grid, env, SourceSpec((50.0,), 75.0), RunOptions(output_stride=1)), 50.0)
    tl = res.tl_field[:, 0, round(75.0 / grid.delta_z)]
    r = res.ranges
    diffs = []
    for i, ri in enumerate(r):
        if 20 * 30.0 <= ri <= grid.max_range / 2:
            j = int(round((2 * ri - r[0]) / grid.delta_r))
            if j < len(r) and abs(r[j] - 2 * ri) < 1e-6:
                diffs.append(tl[j] - tl[i])
    assert abs(np.mean(diffs) - 3.01) <= 0.5


def test_criterion_06_convergence_order():
    def run(dr, n):
        grid = make_grid(n_range=n, n_azimuth=8, n_depth=128, delta_r=dr, delta_z=3.0, r_start=10.0)
        env = make_env(grid)
        l = np.arange(128)
        modes = sum(a * np.sin(q * math.pi * l / 128) for q, a in ((2, 1.0), (3, 0.6), (5, 0.3)))
        az = 1.0 + 0.3 * np.cos(np.arange(8) * grid.delta_theta)
        v = np.outer(az, modes).astype(np.complex128)
        k0 = wavenumber(50.0, 1500.0)
        local = np.ascontiguousarray(O_local(env, grid, k0))
        out = np.empty_like(v)
        g = _native.GridParams(1, 8, 128, 0, n, n, 0, 0, dr, grid.delta_theta, 3.0, 10.0, 10.0)
        _native.call("pe3d_march_host", _native.handle(), g,
                     _native.make_coeffs([k0], [StepCoefficients.for_step(k0, dr)]),
                     _native.ptr(local), _native.ptr(v), _native.ptr(out), None, None, None)
        return out
    e1 = np.linalg.norm(run(5.0, 160) - run(2.5, 320))
    e2 = np.linalg.norm(run(2.5, 320) - run(1.25, 640))
    assert math.log2(e1 / e2) >= 1.0


@pytest.mark.parametrize("chains", ["1", "2"])
def test_criterion_07_executor_invariance(monkeypatch, chains):
    """Reference criterion 7 (tests/test_acceptance.py): TL digests are
    bitwise identical for every executor configuration.  Here: workers,
    schedule and intra_threads of frequency_farm, and the number of
    concurrent step chains."""
    import hashlib
    from paper_1711_00005_b200 import frequency_farm
    monkeypatch.setenv("PE3D_CHAINS", chains)
    cfg = configs.build("cfg1", n_range=40, frequencies=(50.0, 65.0, 80.0), output_stride=10)
    digests = set()
    for workers, schedule, intra in [(1, "static", 1), (2, "static", 1), (4, "dynamic", 2), (3, "dynamic", 8)]:
        rep = frequency_farm(cfg, [50.0, 65.0, 80.0], workers=workers, schedule=schedule, intra_threads=intra)
        assert not rep.failures
        h = hashlib.sha256()
        for r in rep.results:
            h.update(np.ascontiguousarray(r.tl_field).tobytes())
        digests.add(h.hexdigest())
    assert len(digests) == 1


def O_local(env, grid, k0):
    from paper_1711_00005_b200.environment import local_term_grid
    return local_term_grid(env, grid, grid.r_start, k0)[0]


def test_linearity_and_rhs_scaling_full_cfg4():
    """Size-independent property at the full cfg4 grid (64 frequencies):
    the march is linear in the starter."""
    cfg = configs.build("cfg4", n_range=5)
    grid = cfg.grid
    freqs = list(cfg.source.frequencies)
    k0s = [wavenumber(f, 1500.0) for f in freqs]
    rng = np.random.default_rng(11)
    F = len(freqs)
    u1 = rng.standard_normal((F, 256, 1024)) + 1j * rng.standard_normal((F, 256, 1024))
    u2 = rng.standard_normal((F, 256, 1024)) + 1j * rng.standard_normal((F, 256, 1024))
    a, b = 0.7 - 1.1j, -2.0 + 0.4j
    local = np.ascontiguousarray(np.stack([O_local(cfg.environment, grid, k0) for k0 in k0s]))
    coeffs = _native.make_coeffs(k0s, [StepCoefficients.for_step(k0, grid.delta_r) for k0 in k0s])

    def march(u):
        out = np.empty_like(u)
        g = _native.GridParams(F, 256, 1024, 0, 5, 5, 0, 0, grid.delta_r, grid.delta_theta, grid.delta_z,
                               grid.r_start, grid.r_start)
        _native.call("pe3d_march_host", _native.handle(), g, coeffs, _native.ptr(local),
                     _native.ptr(np.ascontiguousarray(u)), _native.ptr(out), None, None, None)
        return out
    x1, x2, x12 = march(u1), march(u2), march(a * u1 + b * u2)
    assert rel_l2(x12, a * x1 + b * x2) <= 1e-12


# ------------------------------------------------------------ slab march (cfg5 decomposition)

@pytest.mark.parametrize("nranks", [1, 2, 4])
def test_slab_march_matches_single_gpu_march(nranks):
    """Virtual ranks exercise the azimuth-slab / depth-slab layouts and the
    chunked all-to-all bookkeeping with the real kernels: bitwise equal to the
    undecomposed march (same per-column and per-ring arithmetic)."""
    from paper_1711_00005_b200 import slab_march
    cfg = configs.build("cfg5", n_range=4, output_stride=2)
    grid = cfg.grid
    small = Config(Grid3D(4, 256, 512, grid.delta_r, 2 * math.pi / 256, grid.delta_z, grid.r_start),
                   cfg.environment, SourceSpec((500.0,), 100.0), RunOptions(output_stride=2))
    ref = march_frequencies(small, [500.0])[0]
    got = slab_march(small, 500.0, nranks)
    assert got.final.tobytes() == ref.final_slab.values.tobytes()
    assert got.tl_field.tobytes() == ref.tl_field.tobytes()
    assert got.clamped_samples == ref.clamped_samples


def test_slab_march_real_nccl_one_rank():
    """The NCCL transport of the slab march (dlopen'd libnccl, unique id
    broadcast through torch.distributed, ncclCommInitRank, grouped
    send/recv) with a single rank on one GPU: bitwise the plain march."""
    import torch.distributed as dist
    from paper_1711_00005_b200 import slab
    cfg = configs.build("cfg5", n_range=4, output_stride=2)
    grid = cfg.grid
    small = Config(Grid3D(4, 256, 512, grid.delta_r, 2 * math.pi / 256, grid.delta_z, grid.r_start),
                   cfg.environment, SourceSpec((500.0,), 100.0), RunOptions(output_stride=2))
    ref = march_frequencies(small, [500.0])[0]
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        got = slab.distributed_slab_march(small, 500.0, device=0)
    finally:
        dist.destroy_process_group()
    assert got.final.tobytes() == ref.final_slab.values.tobytes()
    assert got.tl_field.tobytes() == ref.tl_field.tobytes()


@pytest.mark.parametrize("nranks", [2, 4])
def test_slab_march_peer_vs_copy_transport(monkeypatch, nranks):
    """Virtual ranks: the peer-direct (fused) transposes -- sweeps storing
    straight into the other ranks' inputs, counters ordering the sweeps --
    against the device-copy all-to-all, and both bitwise the plain march."""
    from paper_1711_00005_b200 import slab_march
    cfg = configs.build("cfg5", n_range=5, output_stride=2)
    grid = cfg.grid
    small = Config(Grid3D(5, 512, 2048, grid.delta_r, 2 * math.pi / 512, grid.delta_z, grid.r_start),
                   cfg.environment, SourceSpec((500.0,), 300.0), RunOptions(output_stride=2))
    monkeypatch.setenv("PE3D_DEPTH_NO_SPLIT", "1")      # the slab march runs the lock-step cluster depth sweep
    ref = march_frequencies(small, [500.0])[0]
    monkeypatch.delenv("PE3D_DEPTH_NO_SPLIT")
    monkeypatch.delenv("PE3D_SLAB_COPY", raising=False)
    peer = slab_march(small, 500.0, nranks)
    monkeypatch.setenv("PE3D_SLAB_COPY", "1")
    copy = slab_march(small, 500.0, nranks)
    for got in (peer, copy):
        assert got.final.tobytes() == ref.final_slab.values.tobytes()
        assert got.tl_field.tobytes() == ref.tl_field.tobytes()


def test_slab_march_ipc_peer_one_rank(monkeypatch):
    """The IPC entry points of the peer transport (export, all-gather of the
    handles, barrier, pe3d_march_slab_p2p) with one rank: bitwise the plain
    march (with the cluster depth sweep the slab march also runs)."""
    import socket
    import torch.distributed as dist
    from paper_1711_00005_b200 import slab
    cfg = configs.build("cfg5", n_range=4, output_stride=2)
    grid = cfg.grid
    small = Config(Grid3D(4, 256, 2048, grid.delta_r, 2 * math.pi / 256, grid.delta_z, grid.r_start),
                   cfg.environment, SourceSpec((500.0,), 300.0), RunOptions(output_stride=2))
    monkeypatch.setenv("PE3D_DEPTH_NO_SPLIT", "1")
    ref = march_frequencies(small, [500.0])[0]
    monkeypatch.delenv("PE3D_DEPTH_NO_SPLIT")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        got = slab.distributed_slab_march(small, 500.0, device=0, transport="peer")
    finally:
        dist.destroy_process_group()
    assert got.final.tobytes() == ref.final_slab.values.tobytes()
    assert got.tl_field.tobytes() == ref.tl_field.tobytes()


def test_slab_march_cfg5_full_size_vs_reference(golden):
    from paper_1711_00005_b200 import slab_march
    fx = golden("cfg5_f500_3steps.npz")
    cfg = configs.build("cfg5", n_range=3, output_stride=1)
    r = slab_march(cfg, 500.0, 4)
    u = r.final
    got = u[fx["mi"], fx["li"]]
    assert np.linalg.norm(got - fx["samples"][2]) <= FIELD_TOL * np.linalg.norm(fx["samples"][2])
    assert abs(np.linalg.norm(u) - fx["norms"][2]) <= FIELD_TOL * fx["norms"][2]


@pytest.mark.parametrize("name", ["cfg4", "cfg3"])
def test_starter_column_flag_bitwise_equal_to_slab(name):
    """PE3D_FLAG_STARTER_COLUMN (u0 as one depth column per frequency, what the
    drop-in passes for the reference's azimuth-independent Gaussian starter,
    ref environment.py:270-284) against the full [F][n_theta][n_depth] slab:
    bitwise equal TL, final slabs and clamped counts -- the range-independent
    march and the device-medium march."""
    from paper_1711_00005_b200.environment import gaussian_starter, gaussian_starter_column
    from paper_1711_00005_b200.marching import _grid_params, _local_column
    freqs = (50.0, 130.0) if name == "cfg4" else (25.0,)
    cfg = configs.build(name, n_range=7, frequencies=freqs, output_stride=3)
    grid, env, source, _ = cfg
    k0s = [wavenumber(f, env.c0) for f in freqs]
    coeffs = _native.make_coeffs(k0s, [StepCoefficients.for_step(k0, grid.delta_r) for k0 in k0s])
    F, NT, NZ, S = len(freqs), grid.n_azimuth, grid.n_depth, 1 + 7 // 3
    slab = np.ascontiguousarray(np.stack([gaussian_starter(grid, source, k0).values for k0 in k0s]))
    cols = np.ascontiguousarray(np.stack([gaussian_starter_column(grid, source, k0) for k0 in k0s]))
    out = []
    for u0, flags in ((slab, 0), (cols, _native.FLAG_STARTER_COLUMN)):
        tl = np.empty((F, S, NT, NZ))
        fin = np.empty((F, NT, NZ), dtype=np.complex128)
        cl = np.zeros(F, dtype=np.int64)
        g = _grid_params(grid, F, 7, 3, 0, grid.r_start, flags)
        if name == "cfg4":
            local = np.ascontiguousarray(np.stack([_local_column(env, grid, grid.r_start, k0) for k0 in k0s]))
            _native.call("pe3d_march_host", _native.handle(), g, coeffs, _native.ptr(local), _native.ptr(u0),
                         _native.ptr(fin), _native.ptr(tl), None, _native.ptr(cl))
        else:
            keep = []
            med = _native.make_medium(env.medium, keep)
            _native.call("pe3d_march_medium_host", _native.handle(), g, coeffs, med, _native.ptr(u0),
                         _native.ptr(fin), _native.ptr(tl), None, _native.ptr(cl))
        out.append((tl, fin, cl))
    for x, y in zip(*out):
        assert x.tobytes() == y.tobytes()


def test_slab_wait_times_out_instead_of_hanging(monkeypatch):
    """A rank that never signals (PE3D_SLAB_TEST_STALL drops one depth-sweep
    signal of the peer-transport slab march): the bounded cross-rank wait
    gives up after PE3D_SLAB_TIMEOUT_MS, later waits return at once, and the
    march fails with a CUDA error instead of hanging the stream."""
    from paper_1711_00005_b200 import slab_march
    from paper_1711_00005_b200.errors import NativeError
    cfg = configs.build("cfg5", n_range=4, output_stride=2)
    grid = cfg.grid
    small = Config(Grid3D(4, 256, 2048, grid.delta_r, 2 * math.pi / 256, grid.delta_z, grid.r_start),
                   cfg.environment, SourceSpec((500.0,), 300.0), RunOptions(output_stride=2))
    monkeypatch.delenv("PE3D_SLAB_COPY", raising=False)
    monkeypatch.setenv("PE3D_SLAB_TEST_STALL", "1")
    monkeypatch.setenv("PE3D_SLAB_TIMEOUT_MS", "300")
    with pytest.raises(NativeError, match="aborted"):
        slab_march(small, 500.0, 2)
    monkeypatch.delenv("PE3D_SLAB_TEST_STALL")
    ok = slab_march(small, 500.0, 2)                     # the handle recovers
    assert np.isfinite(ok.final).all()


def test_singular_payload_is_the_lowest_members_own():
    """Many singular members failing at different pivot rows in different
    tiles: the error names the lowest member AND that member's own pivot
    (ref tridiag.py:274-280) -- the key and its payload are swapped together."""
    rng = np.random.default_rng(11)
    n = 9
    systems = [TriDiagSystem(*O.random_system(rng, n, False)) for _ in range(300)]
    expected = None
    for member, pivot in ((290, 1), (77, 6), (150, 3), (77 + 64, 2), (5 + 128, 8), (9, 4)):
        main = np.asarray(systems[member].main).copy()
        sub = np.asarray(systems[member].sub).copy()
        sup = np.asarray(systems[member].sup).copy()
        # make elimination row `pivot` exactly singular: zero row and off-diagonals feeding it
        main[pivot] = 0.0
        if pivot > 0:
            sub[pivot - 1] = 0.0
        systems[member] = TriDiagSystem(sub, main, sup, systems[member].rhs)
        if expected is None or member < expected[0]:
            expected = (member, pivot)
    batch = SolveBatch.from_systems(systems)
    with pytest.raises(SingularSystemError) as ei:
        solve_batch(batch)
    assert (ei.value.member_index, ei.value.pivot_index) == expected


def test_azimuth_step_error_matches_reference(golden):
    """Hand-built coefficients whose periodic azimuth system the reference's
    Sherman-Morrison solve rejects (diag = 0: StepError(1, "azimuth", member 0)
    caused by SingularSystemError(pivot n-1)) or accepts although degenerate
    (diag = 2 off): the same outcome from the B200 range_step, whose
    circulant sweep leaves the decision to the reference's own pivot checks
    (ref marching.py:124-131, tridiag.py:145-212; fixture from the reference)."""
    fx = golden("azimuth_singular.npz")
    grid = Grid3D(10, 8, 16, 5.0, 2 * math.pi / 8, 4.0, 5.0)
    env = Environment(1500.0, SoundSpeedProfile.uniform(1500.0), 6000.0, Absorber(0.75 * grid.depth_extent, 0.01),
                      grid.depth_extent)
    k0 = float(fx["k0"])
    for tag in ("diag0", "diag2off"):
        cy = complex(fx[f"{tag}_cy"])
        co = StepCoefficients(delta=complex(fx["delta"]), cx_lhs=complex(fx["cx_lhs"]), cx_rhs=complex(fx["cx_rhs"]),
                              cy_lhs=cy, cy_rhs=-cy)
        state = MarchState(FieldSlab(np.ones((8, 16), dtype=complex), grid.r_start), 0, co, env, grid, k0)
        raised, j, member, pivot = (int(x) for x in fx[f"{tag}_error"])
        if raised:
            with pytest.raises(StepError) as info:
                range_step(state)
            e = info.value
            assert (e.range_index, e.sweep, e.member_index) == (j, "azimuth", member)
            assert e.__cause__.pivot_index == pivot
        else:
            with np.errstate(all="ignore"):
                range_step(state)
