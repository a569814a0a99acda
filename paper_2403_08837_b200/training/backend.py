"""Kernel backend: the sm_100a operator library (ref `training/backend.py:13-30`).

Same module protocol as the reference backend (`NAME`, `mlp_value_grad`,
`quad_value_grad`), served by `libcdp_b200.so`.  Names "auto", "compiled"
and "cuda" all select it.  There is deliberately no CPU twin: "python" (or
CYCLICDP_PURE=1) raises instead of silently running on the host, and every
call raises `NativeUnavailable` when the library or a CUDA device is absent.
`kernels` is resolved lazily so that importing the package (plan layer,
tests on CPU) never needs a GPU.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .. import _native as N

DTYPE_CODES = {"fp32": 0, "bf16": 1}


class CudaKernels:
    """Backend module protocol over the C-ABI (host fp64 in, fp64 out)."""

    NAME = "cuda-sm100a"

    def __init__(self, dtype: str = "fp32"):
        self.dtype = dtype

    def mlp_value_grad(self, dims, theta, x, y, labels, loss_kind):
        L = N.lib()
        dims_a = np.ascontiguousarray(dims, dtype=np.int64)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        xa = np.ascontiguousarray(x, dtype=np.float64)
        ya = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
        la = None if labels is None else np.ascontiguousarray(labels, dtype=np.int64)
        grad = np.empty(th.shape[0], dtype=np.float64)
        loss = ctypes.c_double()
        N.check(L.cdp_mlp_value_grad(
            len(dims_a), dims_a.ctypes.data_as(N.c_int64_p), th.ctypes.data_as(N.c_double_p), xa.shape[0],
            xa.ctypes.data_as(N.c_double_p), ya.ctypes.data_as(N.c_double_p) if ya is not None else None,
            la.ctypes.data_as(N.c_int64_p) if la is not None else None, int(loss_kind), DTYPE_CODES[self.dtype],
            ctypes.byref(loss), grad.ctypes.data_as(N.c_double_p)))
        return float(loss.value), grad

    def quad_value_grad(self, a, theta, targets):
        L = N.lib()
        av = np.ascontiguousarray(a, dtype=np.float64)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        ts = np.ascontiguousarray(targets, dtype=np.float64)
        grad = np.empty(av.shape[1], dtype=np.float64)
        loss = ctypes.c_double()
        N.check(L.cdp_quad_value_grad(av.shape[0], av.shape[1], av.ctypes.data_as(N.c_double_p),
                                      th.ctypes.data_as(N.c_double_p), ts.shape[0], ts.ctypes.data_as(N.c_double_p),
                                      ctypes.byref(loss), grad.ctypes.data_as(N.c_double_p)))
        return float(loss.value), grad


def load_backend(name: str | None = None):
    if name is None:
        name = "python" if os.environ.get("CYCLICDP_PURE") == "1" else "auto"
    if name in ("auto", "compiled", "cuda"):
        return CudaKernels()
    if name == "python":
        raise N.NativeUnavailable("there is no CPU twin of the sm_100a kernels (no CPU fallback by design)")
    raise ValueError(f"unknown backend {name!r}")


kernels = CudaKernels()
BACKEND_NAME = kernels.NAME
