"""The C ABI surface: the library loads and exports every declared symbol.

Runs without a GPU: no compute calls, only symbol resolution and the error
path (creating a context without a device must fail loudly, never fall back).
"""

import ctypes
import os
import re

import pytest

from paper_2105_10439_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "cofem_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cofem_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_the_binding_expects():
    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_abi_version():
    assert _lib.load().cofem_abi_version() == 1


def test_no_silent_cpu_fallback_without_gpu():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.CofemError):
        _lib.Context(8, 16)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "absent.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load()
