"""libcdp_b200.so loads and exports every symbol include/cdp_b200.h declares (CPU, no GPU calls)."""

import os
import re

import pytest

from paper_2403_08837_b200 import _native


def _declared():
    src = open(_native.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cdp_[a-z0-9_]+)\s*\(", src)))


def test_header_and_bindings_agree():
    assert set(_declared()) == set(_native.SIGNATURES)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libcdp_b200.so not built")
    L = _native.load_library()
    for name in _declared():
        assert hasattr(L, name), name
    assert L.cdp_version() >= 1


def test_no_cpu_fallback():
    from paper_2403_08837_b200.training import load_backend

    with pytest.raises(_native.NativeUnavailable):
        load_backend("python")
