"""CPU checks of the C-ABI boundary: the library loads and exports every symbol
include/qtt.h declares, and the ctypes binding covers exactly those symbols."""
import ctypes
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "qtt.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qtt_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_nonempty():
    syms = declared_symbols()
    assert "qtt_local_matvec" in syms and "qtt_ctx_create" in syms


def test_library_exports_every_declared_symbol():
    from paper_2501_12151_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libqtt.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_matches_header():
    from paper_2501_12151_b200 import _native
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_no_device_fails_loudly():
    """Without a GPU the engine must raise, never fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2501_12151_b200 import _native
    from paper_2501_12151_b200.errors import DeviceError
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libqtt.so not built")
    with pytest.raises(DeviceError):
        _native.Context(0)
