"""ctypes binding of libcdp_b200.so (declarations mirror include/cdp_b200.h).

There is no CPU fallback: `lib()` raises `NativeUnavailable` when the library
is missing or no CUDA device is visible, and every caller propagates it.
"""

from __future__ import annotations

import ctypes
import sys
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CDP_LIB_PATH: an alternative build of the same library (A/B timing of two builds in one process pool)
LIB_PATH = os.environ.get("CDP_LIB_PATH") or os.path.join(HERE, "libcdp_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "cdp_b200.h")

c_int, c_float, c_double, c_void_p, c_size_t = ctypes.c_int, ctypes.c_float, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_double_p = ctypes.POINTER(ctypes.c_double)
c_float_p = ctypes.POINTER(ctypes.c_float)
c_int_p = ctypes.POINTER(ctypes.c_int)
c_u8_p = ctypes.POINTER(ctypes.c_uint8)

# name -> (restype, argtypes); kept in the header's order.
SIGNATURES = {
    "cdp_last_error": (ctypes.c_char_p, []),
    "cdp_version": (c_int, []),
    "cdp_device_sm_count": (c_int, []),
    "cdp_set_device": (c_int, [c_int]),
    "cdp_memcpy_d2h": (c_int, [c_void_p, c_void_p, c_size_t]),
    "cdp_mlp_value_grad": (c_int, [c_int, c_int64_p, c_double_p, c_int, c_double_p, c_double_p, c_int64_p, c_int,
                                   c_int, c_double_p, c_double_p]),
    "cdp_quad_value_grad": (c_int, [c_int, c_int, c_double_p, c_double_p, c_int, c_double_p, c_double_p, c_double_p]),
    "cdp_trainer_create": (c_int, [c_int, c_int64_p, c_int, c_int, c_int, c_int, c_float, c_float, c_int,
                                   ctypes.POINTER(ctypes.c_int32), c_int, ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32), c_int, c_float_p, ctypes.POINTER(ctypes.c_int32),
                                   c_float_p, ctypes.POINTER(c_void_p)]),
    "cdp_trainer_destroy": (None, [c_void_p]),
    "cdp_trainer_create_rank": (c_int, [c_int, c_int64_p, c_int, c_int, c_int, c_int, c_int, c_float, c_float, c_int,
                                        ctypes.POINTER(ctypes.c_int32), c_int, c_float_p,
                                        ctypes.POINTER(ctypes.c_int32), c_float_p, ctypes.POINTER(c_void_p)]),
    "cdp_trainer_region": (c_int, [c_void_p, ctypes.POINTER(c_void_p), ctypes.POINTER(c_size_t)]),
    "cdp_trainer_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "cdp_ipc_open": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "cdp_ipc_close": (c_int, [c_void_p]),
    "cdp_trainer_connect": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "cdp_trainer_ring_error": (c_int, [c_void_p, c_int_p]),
    "cdp_trainer_partial": (c_int, [c_void_p, ctypes.POINTER(c_void_p), ctypes.POINTER(c_size_t)]),
    "cdp_trainer_apply_update": (c_int, [c_void_p]),
    "cdp_trainer_set_params": (c_int, [c_void_p, c_int, c_float_p]),
    "cdp_trainer_get_params": (c_int, [c_void_p, c_int, c_float_p]),
    "cdp_trainer_set_velocity": (c_int, [c_void_p, c_float_p]),
    "cdp_trainer_get_velocity": (c_int, [c_void_p, c_float_p]),
    "cdp_trainer_step": (c_int, [c_void_p, ctypes.POINTER(ctypes.c_int32), c_float]),
    "cdp_trainer_step_host_batch": (c_int, [c_void_p, c_float_p, ctypes.POINTER(ctypes.c_int32), c_float_p, c_float]),
    "cdp_trainer_sync": (c_int, [c_void_p]),
    "cdp_trainer_history": (c_int, [c_void_p, c_int, c_double_p, ctypes.POINTER(ctypes.c_uint32), c_int_p]),
    "cdp_trainer_stats": (c_int, [c_void_p, c_int64_p, c_int]),
    "cdp_trainer_get_grad": (c_int, [c_void_p, c_float_p]),
    "cdp_trainer_last": (c_int, [c_void_p, c_double_p, ctypes.POINTER(ctypes.c_uint32)]),
    "cdp_trainer_time_op": (c_int, [c_void_p, c_int, c_int, c_int, c_float_p]),
    "cdp_trainer_mark": (c_int, [c_void_p, c_int]),
    "cdp_trainer_elapsed": (c_int, [c_void_p, c_int, c_int, c_float_p]),
    "cdp_trainer_flush_l2": (c_int, [c_void_p]),
    "cdp_trainer_set_trace": (c_int, [c_void_p, c_int]),
    "cdp_trainer_trace": (c_int, [c_void_p, ctypes.POINTER(ctypes.c_uint64), c_int]),
    "cdp_trainer_stream": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "cdp_resnet_create_rank": (c_int, [c_int, c_int_p, c_int_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                       c_int, c_int, c_int_p, c_u8_p, c_int, c_float, c_float, c_int, c_float_p,
                                       c_int_p, c_int_p, c_int, ctypes.POINTER(c_void_p)]),
    "cdp_resnet_zero_drain": (c_int, [c_void_p]),
    "cdp_resnet_zero_state": (c_int, [c_void_p, c_int, c_float_p, ctypes.POINTER(ctypes.c_uint32)]),
    "cdp_resnet_zero_drain_plan": (c_int, [c_void_p, ctypes.POINTER(ctypes.c_int32), c_int]),
    "cdp_resnet_pull_chain": (c_int, [c_void_p, ctypes.POINTER(ctypes.c_int32), c_int]),
    "cdp_resnet_apply_update": (c_int, [c_void_p]),
    "cdp_resnet_apply_update_range": (c_int, [c_void_p, c_int, c_int]),
    "cdp_resnet_pack_range": (c_int, [c_void_p, c_int, c_int, c_int]),
    "cdp_resnet_partial": (c_int, [c_void_p, ctypes.POINTER(c_void_p), ctypes.POINTER(ctypes.c_size_t)]),
    "cdp_resnet_stream": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "cdp_resnet_step_host_batch": (c_int, [c_void_p, c_float_p, c_int_p, c_float]),
    "cdp_resnet_step_host_batch_async": (c_int, [c_void_p, c_float_p, c_int_p, c_float, c_int]),
    "cdp_resnet_last_loss": (c_int, [c_void_p, c_double_p]),
    "cdp_resnet_profile_step": (c_int, [c_void_p, c_int_p, c_float, c_int, c_int, ctypes.c_char_p, c_int, c_double_p,
                                        c_double_p, c_float_p, c_int_p]),
    "cdp_resnet_info": (c_int, [c_void_p, c_int64_p, c_int_p, c_int64_p, c_int_p]),
    "cdp_resnet_region": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "cdp_resnet_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "cdp_resnet_connect": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "cdp_resnet_destroy": (None, [c_void_p]),
    "cdp_resnet_set_params": (c_int, [c_void_p, c_int, c_float_p]),
    "cdp_resnet_get_params": (c_int, [c_void_p, c_int, c_float_p]),
    "cdp_resnet_step": (c_int, [c_void_p, c_int_p, c_float]),
    "cdp_resnet_history": (c_int, [c_void_p, c_int, c_double_p, ctypes.POINTER(ctypes.c_uint32), c_int_p]),
    "cdp_resnet_sync": (c_int, [c_void_p]),
    "cdp_resnet_ring_error": (c_int, [c_void_p, c_int_p]),
    "cdp_resnet_stats": (c_int, [c_void_p, c_int64_p, c_int]),
    "cdp_resnet_mark": (c_int, [c_void_p, c_int]),
    "cdp_resnet_elapsed": (c_int, [c_void_p, c_int, c_int, c_float_p]),
    "cdp_resnet_flush_l2": (c_int, [c_void_p]),
    "cdp_resnet_trace": (c_int, [c_void_p, ctypes.POINTER(ctypes.c_uint32), c_int, c_int_p]),
    "cdp_resnet_buffer": (c_int, [c_void_p, ctypes.c_char_p, c_int, ctypes.POINTER(c_void_p),
                                  ctypes.POINTER(c_size_t), c_int_p]),
    "cdp_vit_create_rank": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int_p,
                                    c_u8_p, c_float, c_float, c_int, c_float_p, c_int_p, c_int,
                                    ctypes.POINTER(c_void_p)]),
    "cdp_vit_create_cyclic": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int_p, c_u8_p,
                                      c_int, c_int_p, c_int_p, c_int_p, c_float, c_float, c_int, c_int, c_float_p,
                                      c_int_p, c_int, ctypes.POINTER(c_void_p)]),
    "cdp_vit_info": (c_int, [c_void_p, c_int64_p, c_int_p]),
    "cdp_vit_set_trace": (c_int, [c_void_p, c_int]),
    "cdp_vit_trace": (c_int, [c_void_p, ctypes.POINTER(ctypes.c_uint32), c_int, c_int_p]),
    "cdp_vit_region": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "cdp_vit_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "cdp_vit_connect": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "cdp_vit_destroy": (None, [c_void_p]),
    "cdp_vit_set_params": (c_int, [c_void_p, c_int, c_float_p]),
    "cdp_vit_get_params": (c_int, [c_void_p, c_int, c_float_p]),
    "cdp_vit_step": (c_int, [c_void_p, c_int_p, c_float]),
    "cdp_vit_step_host_batch": (c_int, [c_void_p, c_float_p, c_int_p, c_float]),
    "cdp_vit_profile_step": (c_int, [c_void_p, c_int_p, c_float, c_int, c_int, ctypes.c_char_p, c_int, c_double_p,
                                     c_double_p, c_float_p, c_int_p]),
    "cdp_vit_history": (c_int, [c_void_p, c_int, c_double_p, ctypes.POINTER(ctypes.c_uint32), c_int_p]),
    "cdp_vit_sync": (c_int, [c_void_p]),
    "cdp_vit_ring_error": (c_int, [c_void_p, c_int_p]),
    "cdp_vit_stats": (c_int, [c_void_p, c_int64_p, c_int]),
    "cdp_vit_mark": (c_int, [c_void_p, c_int]),
    "cdp_vit_elapsed": (c_int, [c_void_p, c_int, c_int, c_float_p]),
    "cdp_vit_flush_l2": (c_int, [c_void_p]),
    "cdp_vit_pull_chain": (c_int, [c_void_p, ctypes.POINTER(ctypes.c_int32), c_int]),
    "cdp_attention": (c_int, [c_void_p, ctypes.c_int64, c_void_p, ctypes.c_int64, c_int, c_int, c_int, c_void_p,
                              ctypes.c_int64, c_void_p, c_void_p, ctypes.c_int64, c_int]),
    "cdp_test_gemm": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(c_void_p), c_int,
                              ctypes.POINTER(c_void_p), c_int, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
}


class NativeUnavailable(RuntimeError):
    pass


class NativeError(RuntimeError):
    pass


_lib = None


def load_library(path: str = LIB_PATH):
    """dlopen + bind signatures; does not require a GPU (used by CPU tests)."""
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} not built: run `python -m paper_2403_08837_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


def lib():
    global _lib
    if _lib is None:
        L = load_library()
        _bind_device(L)
        if L.cdp_device_sm_count() <= 0:
            raise NativeUnavailable("no CUDA device visible to libcdp_b200 (the sm_100a path has no CPU fallback)")
        _lib = L
    else:
        _bind_device(_lib)
    return _lib


def _bind_device(L):
    """The library links its own CUDA runtime: select torch's current device for this thread (one process
    per GPU: the rank's torch.cuda.set_device(LOCAL_RANK) then also places the trainers)."""
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        if L.cdp_set_device(int(torch.cuda.current_device())) != 0:
            raise NativeError(L.cdp_last_error().decode())


def check(rc: int) -> None:
    if rc != 0:
        raise NativeError(lib().cdp_last_error().decode())


def memcpy_d2h(dst: int, src: int, nbytes: int) -> None:
    check(lib().cdp_memcpy_d2h(ctypes.c_void_p(dst), ctypes.c_void_p(src), nbytes))


TRACE_FIELDS = ("t", "rank", "unit", "kind", "phase", "slot", "version")


def read_access_trace(fn, handle, max_records=1 << 16):
    """Executed-version records of a trace-mode trainer (cdp_resnet_trace / cdp_vit_trace): structured array
    with fields t, rank, unit (1-based), kind (0 fwd / 1 bwd / 2 update read / 3 update's new slot),
    phase (0 before / 1 after), slot, version (the tag of the data found in the slot)."""
    import numpy as np

    buf = np.zeros((max_records, 8), dtype=np.uint32)
    n = ctypes.c_int()
    check(fn(handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), max_records, ctypes.byref(n)))
    if n.value > max_records:
        raise RuntimeError(f"{n.value} trace records, read at most {max_records}")
    r = buf[: n.value].astype(np.int64)
    out = np.empty(n.value, dtype=np.dtype([(k, np.int64) for k in TRACE_FIELDS]))
    for i, k in enumerate(TRACE_FIELDS):
        out[k] = r[:, i]
    return out
