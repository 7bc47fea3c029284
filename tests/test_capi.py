"""CPU suite: the C-ABI library loads and exports every symbol the header declares."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fraclap_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fl_\w+)\s*\(", txt)))


def test_header_and_binding_agree():
    from paper_1809_01971_b200 import _lib
    assert header_symbols() == _lib.exported_symbols()


def test_library_exports_every_symbol():
    from paper_1809_01971_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libfraclap_b200.so not built")
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.fl_version() == 1


def test_no_cuda_fails_loudly():
    import torch
    from paper_1809_01971_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError):
        _lib.require_cuda()
