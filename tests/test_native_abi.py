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


def test_library_follows_torch_current_device(monkeypatch):
    """The library links its own CUDA runtime; lib() binds it to torch's current device (one process per
    GPU: the rank's torch.cuda.set_device(LOCAL_RANK) places the trainers) and leaves it alone when torch
    has not initialised CUDA."""
    import torch

    calls = []

    class FakeLib:
        def cdp_set_device(self, d):
            calls.append(d)
            return 0

        def cdp_last_error(self):
            return b""

    monkeypatch.setattr(torch.cuda, "is_initialized", lambda: False)
    _native._bind_device(FakeLib())
    assert calls == []
    monkeypatch.setattr(torch.cuda, "is_initialized", lambda: True)
    monkeypatch.setattr(torch.cuda, "current_device", lambda: 3)
    _native._bind_device(FakeLib())
    assert calls == [3]
