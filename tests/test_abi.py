"""The C-ABI library loads and exports every symbol include/piecy_b200.h
declares (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "piecy_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pcy_[a-z0-9_]+)\s*\(", txt)))


def test_header_lists_the_api():
    syms = header_symbols()
    for must in ("pcy_engine_create", "pcy_engine_insert", "pcy_engine_extract", "pcy_kmeanspp",
                 "pcy_lloyd", "pcy_rsvd", "pcy_project", "pcy_last_error"):
        assert must in syms


def test_library_exports_every_header_symbol():
    from paper_1502_04265_b200 import _build
    path = _build.build()
    lib = ctypes.CDLL(path)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_1502_04265_b200 import _native, evaluation, linalg  # noqa: F401  (register symbols)
    syms = header_symbols()
    bound = set(_native._SIGS)
    assert not [s for s in syms if s not in bound]


def test_no_gpu_means_loud_failure():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_1502_04265_b200 import BicoEngine
    from paper_1502_04265_b200._native import NativeError
    with pytest.raises(NativeError):
        BicoEngine(3, 10)
