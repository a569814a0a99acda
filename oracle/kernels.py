"""ORACLE — TEST INFRASTRUCTURE ONLY.  ctypes front of `cdp_oracle.c` and a
loader for the reference's compiled kernel in `oracle/_ref/`.

Same call signatures as the reference backend module protocol
(`pkg/src/cyclicdp/training/backend.py:13-30`): `mlp_value_grad(dims, theta,
x, y, labels, loss_kind) -> (loss, grad)` and `quad_value_grad(a, theta,
targets) -> (loss, grad)`, all fp64.
"""

from __future__ import annotations

import ctypes
import importlib.util
import os

import numpy as np

from . import build as _build

NAME = "oracle-c"

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.LIB
        if not os.path.exists(path):
            _build.build_oracle()
        L = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        L.oracle_mlp_value_grad.restype = ctypes.c_double
        L.oracle_mlp_value_grad.argtypes = [ctypes.c_int, ip, dp, ctypes.c_int, dp, dp, ip, ctypes.c_int, dp]
        L.oracle_quad_value_grad.restype = ctypes.c_double
        L.oracle_quad_value_grad.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, ctypes.c_int, dp, dp]
        L.oracle_mlp_value_grad_batch.restype = None
        pp = ctypes.POINTER(dp)
        L.oracle_mlp_value_grad_batch.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, pp, ctypes.c_int, pp, pp,
            ctypes.POINTER(ip), ctypes.c_int, pp, dp,
        ]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def mlp_value_grad(dims, theta, x, y, labels, loss_kind):
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    xa = np.ascontiguousarray(x, dtype=np.float64)
    ya = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    la = None if labels is None else np.ascontiguousarray(labels, dtype=np.int64)
    grad = np.empty(th.shape[0], dtype=np.float64)
    loss = lib().oracle_mlp_value_grad(
        len(dims_a), _i(dims_a), _d(th), xa.shape[0], _d(xa),
        _d(ya) if ya is not None else None, _i(la) if la is not None else None, int(loss_kind), _d(grad),
    )
    return float(loss), grad


def mlp_value_grad_many(dims, thetas, xs, labels, loss_kind, threads):
    """Several independent micro-batches at once (pthreads), xent/labels or mse/ys."""
    n = len(xs)
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    ths = [np.ascontiguousarray(t, dtype=np.float64) for t in thetas]
    xa = [np.ascontiguousarray(x, dtype=np.float64) for x in xs]
    grads = [np.empty(ths[0].shape[0]) for _ in range(n)]
    losses = np.empty(n)
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int64)
    if loss_kind == 1:
        la = [np.ascontiguousarray(l, dtype=np.int64) for l in labels]
        lab_arr = (ip * n)(*[_i(l) for l in la])
        y_arr = None
    else:
        la = [np.ascontiguousarray(l, dtype=np.float64) for l in labels]
        y_arr = (dp * n)(*[_d(l) for l in la])
        lab_arr = None
    lib().oracle_mlp_value_grad_batch(
        n, int(threads), len(dims_a), _i(dims_a), (dp * n)(*[_d(t) for t in ths]), xa[0].shape[0],
        (dp * n)(*[_d(x) for x in xa]), y_arr, lab_arr, int(loss_kind), (dp * n)(*[_d(g) for g in grads]),
        _d(losses),
    )
    return [float(l) for l in losses], grads


def quad_value_grad(a, theta, targets):
    av = np.ascontiguousarray(a, dtype=np.float64)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    ts = np.ascontiguousarray(targets, dtype=np.float64)
    grad = np.empty(av.shape[1])
    loss = lib().oracle_quad_value_grad(av.shape[0], av.shape[1], _d(av), _d(th), ts.shape[0], _d(ts), _d(grad))
    return float(loss), grad


def load_reference_kernels():
    """The reference's own compiled `_kernels` module from oracle/_ref, or None."""
    path = _build.ref_module_path()
    if not os.path.exists(path):
        path = _build.build_ref()
        if path is None or not os.path.exists(path):
            return None
    spec = importlib.util.spec_from_file_location("_kernels", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
