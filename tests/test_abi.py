"""The C-ABI library loads and exports every symbol include/pe3d_b200.h
declares; without a GPU the compute path fails loudly (no CPU fallback)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_1711_00005_b200 import _native, errors

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pe3d_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"PE3D_API\s+\w+\s+(pe3d_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pe3d_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_version_and_sample_count():
    lib = _native.load_library()
    assert lib.pe3d_abi_version() == _native.ABI_VERSION
    assert lib.pe3d_sample_count(400, 10) == 41
    assert lib.pe3d_sample_count(0, 3) == 1
    assert lib.pe3d_sample_count(5, 0) == -1


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly():
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(errors.NativeError):
        _native.handle(0)


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(errors.NativeError, match="missing"):
        _native.load_library(tmp_path / "nope.so")
