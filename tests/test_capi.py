"""The C-ABI library loads and exports every symbol include/sgad.h declares
(no GPU needed: loading does not touch the device)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sgad.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sgad_\w+)\s*\(", src, re.M)))


def test_header_declares_api():
    syms = declared_symbols()
    assert "sgad_raster_prepare" in syms and "sgad_track_normal_eqs" in syms
    assert len(syms) >= 19


def test_library_exports_every_declared_symbol():
    from paper_2603_21055_b200 import _native
    from paper_2603_21055_b200.build import build
    lib_path = build()
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(_native.EXPORTS)
    lib.sgad_version.restype = ctypes.c_int
    assert lib.sgad_version() == 1


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2603_21055_b200 import _native
    with pytest.raises(RuntimeError, match="CUDA"):
        _native.load()
