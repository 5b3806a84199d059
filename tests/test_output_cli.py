"""On-disk formats and the INI/CLI front end.

The TL CSV / binary grid / manifest writers must produce the same bytes as
the reference's (fixtures written by the reference itself:
tests/golden/make_golden.py output)."""

import math
import subprocess
import sys

import numpy as np
import pytest

from paper_1711_00005_b200 import FieldSlab, FrequencyResult, Grid3D
from paper_1711_00005_b200 import output as out
from paper_1711_00005_b200.config import load_config
from paper_1711_00005_b200.errors import ConfigError, InvariantError

from conftest import GOLDEN, ROOT


def fixture_result():
    fx = np.load(GOLDEN / "output" / "inputs.npz")
    grid = Grid3D(10, 4, 5, 5.0, 2 * math.pi / 4, 3.0, 5.0)
    rng = np.random.default_rng(0)
    res = FrequencyResult(frequency=63.5, ranges=fx["ranges"], tl_field=fx["tl"], clamped_samples=1,
                          final_slab=FieldSlab(rng.standard_normal((4, 5)), 25.0), output_stride=2,
                          wall_seconds=0.5)
    return res, grid


def test_csv_bytes_match_reference(tmp_path):
    res, grid = fixture_result()
    p = out.write_tl_csv(tmp_path / "tl.csv", res, grid)
    assert p.read_bytes() == (GOLDEN / "output" / "ref_tl.csv").read_bytes()
    meta, tl = out.read_tl_csv(p)
    assert meta["n_depth"] == "5" and np.allclose(tl, res.tl_field, atol=1e-6)


def test_binary_bytes_match_reference(tmp_path):
    res, grid = fixture_result()
    p = out.write_tl_binary(tmp_path / "tl.bin", res, grid)
    assert p.read_bytes() == (GOLDEN / "output" / "ref_tl.bin").read_bytes()
    meta, tl = out.read_tl_binary(p)
    assert meta["ranges_m"] == [5.0, 15.0, 25.0] and np.array_equal(tl, res.tl_field)


def test_manifest_bytes_match_reference(tmp_path):
    out.write_manifest(tmp_path, {"command": "run", "frequencies": [{"frequency_hz": 63.5, "sha256": "x"}],
                                  "grid": {"n_range": 10}})
    assert (tmp_path / out.MANIFEST_NAME).read_bytes() == (GOLDEN / "output" / out.MANIFEST_NAME).read_bytes()
    assert out.load_manifest(tmp_path)["grid"]["n_range"] == 10


def test_filename_and_format_rules(tmp_path):
    assert out.tl_filename(63.5, "csv") == "tl_0000063.5000Hz.csv"
    assert out.tl_filename(500, "binary-grid") == "tl_0000500.0000Hz.bin"
    res, grid = fixture_result()
    with pytest.raises(InvariantError):
        out.write_tl_grid(tmp_path / "x", res, grid, "hdf5")
    bad = FrequencyResult(63.5, res.ranges, res.tl_field * np.nan, 0, res.final_slab, 2, 0.0)
    with pytest.raises(InvariantError, match="finite"):
        out.write_tl_csv(tmp_path / "y.csv", bad, grid)
    (tmp_path / "z.bin").write_bytes(b"NOTAGRID" + b"\0" * 8)
    with pytest.raises(ConfigError):
        out.read_tl_binary(tmp_path / "z.bin")


REFERENCE_INI = """\
[grid]
n_range = 50
n_azimuth = 360
n_depth = 512
delta_r = 10.0
delta_theta = 1.0
delta_z = 4.0
r_start = 10.0

[environment]
c0 = 1500.0
sound_speed = 1500.0
water_depth = 6000.0
absorber_start_depth = 1500.0
absorber_max_attenuation = 0.01

[source]
frequencies = 25.0, 40.0, 50.0, 63.0
depth = 100.0

[run]
output_stride = 10
tl_format = binary-grid
"""


def test_reference_ini_parses(tmp_path):
    p = tmp_path / "medium.ini"
    p.write_text(REFERENCE_INI)
    c = load_config(p)
    assert (c.grid.n_range, c.grid.n_azimuth, c.grid.n_depth) == (50, 360, 512)
    assert c.grid.delta_theta == math.radians(1.0) and c.grid.r_start == 10.0
    assert c.environment.absorber.start_depth == 1500.0 and c.environment.medium is None
    assert c.source.frequencies == (25.0, 40.0, 50.0, 63.0)
    assert c.options.output_stride == 10 and c.options.tl_format == "binary-grid"


def test_extended_medium_section(tmp_path):
    p = tmp_path / "cfg.ini"
    p.write_text(REFERENCE_INI.replace("[source]", """[medium]
bottom_speed = 1700
bottom_density = 1.5
bottom_alpha = 0.5
bathymetry_depth = 150
sponge_points = 32

[source]"""))
    c = load_config(p)
    m = c.environment.medium
    assert m.bottom.speed == 1700 and m.bottom.density == 1.5 and m.sponge.n_points == 32
    assert m.range_independent


def test_ini_errors(tmp_path):
    p = tmp_path / "bad.ini"
    p.write_text("[grid]\nn_range = x\n")
    with pytest.raises(ConfigError):
        load_config(p)
    p.write_text(REFERENCE_INI.replace("n_azimuth = 360", "n_azimuth = abc"))
    with pytest.raises(ConfigError, match="n_azimuth"):
        load_config(p)
    with pytest.raises(ConfigError, match="not found"):
        load_config(tmp_path / "missing.ini")


def test_cli_config_error_exit_code(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_1711_00005_b200", "run", "--config", str(tmp_path / "no.ini")],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 2 and "config error" in r.stderr


@pytest.mark.gpu
def test_cli_run_end_to_end(tmp_path):
    from oracle import pe3d_oracle as O
    p = tmp_path / "run.ini"
    p.write_text(REFERENCE_INI.replace("n_range = 50", "n_range = 20"))
    r = subprocess.run([sys.executable, "-m", "paper_1711_00005_b200", "run", "--config", str(p),
                        "--output", str(tmp_path / "o")], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    man = out.load_manifest(tmp_path / "o")
    assert [e["status"] for e in man["frequencies"]] == ["ok"] * 4
    for e in man["frequencies"]:
        assert out.file_sha256(tmp_path / "o" / e["file"]) == e["sha256"]
    meta, tl = out.read_tl_binary(tmp_path / "o" / man["frequencies"][2]["file"])
    ref = O.run_frequency(load_config(p), 50.0)
    mask = ref.tl_field < 150
    assert np.abs(tl - ref.tl_field)[mask].max() <= 1e-4
