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


def test_call_retries_once_after_scratch_oom(monkeypatch):
    """_lib.call: FL_ENOMEM (the library's stream-ordered scratch lost the race
    for device memory against torch's cache) empties torch's cache and retries
    once; a second failure surfaces as FraclapError."""
    from paper_1809_01971_b200 import _lib

    class Fake:
        def __init__(self, codes):
            self.codes = list(codes)
            self.calls = 0

        def fl_thing(self, *args):
            self.calls += 1
            return self.codes.pop(0)

        def fl_last_error(self):
            return b"cudaMallocAsync: out of memory"

    fake = Fake([_lib.FL_ENOMEM, _lib.FL_OK])
    monkeypatch.setattr(_lib, "load", lambda: fake)
    _lib.call("fl_thing", 1, 2)
    assert fake.calls == 2
    fake = Fake([_lib.FL_ENOMEM, _lib.FL_ENOMEM])
    monkeypatch.setattr(_lib, "load", lambda: fake)
    with pytest.raises(_lib.FraclapError):
        _lib.call("fl_thing")
    assert fake.calls == 2
    fake = Fake([_lib.FL_EINVAL])
    monkeypatch.setattr(_lib, "load", lambda: fake)
    with pytest.raises(ValueError):
        _lib.call("fl_thing")
    assert fake.calls == 1
