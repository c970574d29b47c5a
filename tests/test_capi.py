"""The drop-in boundary: libhn.so builds for sm_100a, loads without a GPU and exports
exactly the entry points include/hn.h declares (no compute calls here)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hn.h"


def header_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void)\s+(hn_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2303_01760_b200 import _build
    return _build.build()


def test_header_declares_entry_points():
    syms = header_symbols()
    for must in ("hn_knn", "hn_weights_mon", "hn_weights_rbf", "hn_apply_ell", "hn_momentum", "hn_div_rhs",
                 "hn_correct_temperature", "hn_temperature_bc", "hn_sptrsv_super", "hn_reduce"):
        assert must in syms


def test_library_loads_and_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(str(lib_path))
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_ctypes_table_matches_header(lib_path):
    from paper_2303_01760_b200 import _lib
    declared = set(header_symbols())
    bound = set(_lib.SIGNATURES)
    assert bound == declared


def test_exported_symbols_are_only_the_abi(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True, text=True).stdout
    ours = {line.split()[-1] for line in out.splitlines() if line.split()[-1].startswith("hn_")}
    assert ours == set(header_symbols())


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib_path)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_loud_failure(monkeypatch):
    """Without CUDA the product path raises -- there is no CPU fallback."""
    import torch
    from paper_2303_01760_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    monkeypatch.setattr(_lib, "_torch", None)
    with pytest.raises(_lib.NativeError):
        _lib.torch()
