"""The C-ABI library loads and exports every declared symbol (CPU, no compute)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2506_05229_b200 import _lib
from paper_2506_05229_b200.errors import DeviceError


def header_symbols():
    text = open(os.path.join(ROOT, "include", "armt_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(armt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTS) == declared


def test_abi_struct_layout_matches_binding():
    lib = _lib.load()
    assert lib.armt_abi_sizeof(0) == ctypes.sizeof(_lib.ArmtGemmArgs)
    assert lib.armt_abi_sizeof(1) == ctypes.sizeof(_lib.ArmtMembers)
    assert lib.armt_abi_sizeof(2) == _lib.ArmtGemmArgs.a_slot.offset


def test_introspection_without_gpu():
    lib = _lib.load()
    assert lib.armt_version().startswith(b"armt_b200")
    assert lib.armt_fold_workspace_bytes(16, 128, 384) == 4 * 16 * 128 * 386


def test_validation_errors_map_to_reference_types():
    # argument validation happens before any device work
    from paper_2506_05229_b200.errors import DimensionError, InputError
    args = _lib.ArmtGemmArgs()
    args.G = 0
    with pytest.raises(DimensionError):
        _lib.check(_lib.load().armt_gemm(args, None), "gemm")
    args.G, args.M, args.N, args.K = 1, 4, 4, 4
    with pytest.raises(InputError):
        _lib.check(_lib.load().armt_gemm(args, None), "gemm")


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(DeviceError):
        _lib.load(str(tmp_path / "nope.so"))
