"""Device-resident CDP / DP trainer over the C-ABI (`cdp_trainer_*`).

One `DeviceMlpTrainer` owns the parameter versions (two slots), momentum,
partial-sum buffer, activation-record slots and the two captured step graphs
of one (model, rule, dtype) configuration.  `step()` launches one training
step asynchronously; `history()` returns the per-step mean losses and the
non-finite flags the kernels raised.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .executor import StepPlan, compile_rank_plan, compile_step_plan
from .rules import UpdateRule

DTYPES = {"fp32": 0, "bf16": 1}


def _i32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _f32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


class DeviceMlpTrainer:
    def __init__(self, dims, micro_batch: int, n_workers: int, loss_kind: int, rule: UpdateRule | None,
                 dtype: str = "fp32", momentum: float = 0.0, weight_decay: float = 0.0,
                 inputs: np.ndarray | None = None, targets: np.ndarray | None = None, grad_only: bool = False,
                 layer_stage=None):
        if dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {sorted(DTYPES)}")
        self.lib = N.lib()
        self.dims = tuple(int(d) for d in dims)
        self.n_stages = len(self.dims) - 1
        self.micro_batch = int(micro_batch)
        self.n_workers = int(n_workers)
        self.loss_kind = int(loss_kind)
        self.dtype = dtype
        self.n_layers = len(self.dims) - 1
        if layer_stage is not None:
            self.n_stages = max(layer_stage)
        self.plan: StepPlan = compile_step_plan(self.n_stages, self.n_workers, rule, grad_only=grad_only,
                                                layer_stage=layer_stage)
        self.sizes = [self.dims[j] * self.dims[j + 1] + self.dims[j + 1] for j in range(self.n_layers)]
        self.P = sum(self.sizes)
        dims_a = np.asarray(self.dims, dtype=np.int64)
        n = 0
        x = lab = tgt = None
        if inputs is not None:
            x = np.ascontiguousarray(inputs, dtype=np.float32)
            n = x.shape[0]
            if loss_kind == 1:
                lab = np.ascontiguousarray(targets, dtype=np.int32)
            else:
                tgt = np.ascontiguousarray(targets, dtype=np.float32)
        ops = np.ascontiguousarray(self.plan.ops, dtype=np.int32)
        deps = np.ascontiguousarray(self.plan.deps, dtype=np.int32)
        slots = np.ascontiguousarray(self.plan.slots, dtype=np.int32)
        h = ctypes.c_void_p()
        N.check(self.lib.cdp_trainer_create(
            len(dims_a), dims_a.ctypes.data_as(N.c_int64_p), self.micro_batch, self.n_workers, self.loss_kind,
            DTYPES[dtype], float(momentum), float(weight_decay), ops.shape[0], _i32(ops), deps.shape[0], _i32(deps),
            _i32(slots), n, _f32(x) if x is not None else None, _i32(lab) if lab is not None else None,
            _f32(tgt) if tgt is not None else None, ctypes.byref(h)))
        self.h = h
        self.has_momentum = momentum != 0.0
        self._keep = (x, lab, tgt)

    @classmethod
    def for_rank(cls, dims, micro_batch: int, world: int, rank: int, loss_kind: int, rule: UpdateRule | None,
                 dtype: str = "fp32", momentum: float = 0.0, weight_decay: float = 0.0,
                 inputs: np.ndarray | None = None, targets: np.ndarray | None = None,
                 layer_stage=None, allreduce: bool = False) -> "DeviceMlpTrainer":
        """One rank of multi-GPU CDP (worker rank+1 on this process's GPU); call connect_* next."""
        self = cls.__new__(cls)
        self.lib = N.lib()
        self.dims = tuple(int(d) for d in dims)
        self.n_layers = len(self.dims) - 1
        self.n_stages = world if layer_stage is not None else self.n_layers
        if layer_stage is None and self.n_layers != world:
            raise ValueError("multi-GPU CDP ties stages = micro-batches = ranks (pass layer_stage to group layers)")
        self.micro_batch, self.n_workers, self.loss_kind, self.dtype = int(micro_batch), 1, int(loss_kind), dtype
        self.rank, self.world = rank, world
        self.sizes = [self.dims[j] * self.dims[j + 1] + self.dims[j + 1] for j in range(self.n_layers)]
        self.P = sum(self.sizes)
        self.rank_ops = compile_rank_plan(world, rank, rule, layer_stage, allreduce=allreduce)
        self.plan = None
        dims_a = np.asarray(self.dims, dtype=np.int64)
        x = lab = tgt = None
        n = 0
        if inputs is not None:
            x = np.ascontiguousarray(inputs, dtype=np.float32)
            n = x.shape[0]
            if loss_kind == 1:
                lab = np.ascontiguousarray(targets, dtype=np.int32)
            else:
                tgt = np.ascontiguousarray(targets, dtype=np.float32)
        ops = np.ascontiguousarray(self.rank_ops, dtype=np.int32)
        h = ctypes.c_void_p()
        N.check(self.lib.cdp_trainer_create_rank(
            len(dims_a), dims_a.ctypes.data_as(N.c_int64_p), self.micro_batch, world, rank, self.loss_kind,
            DTYPES[dtype], float(momentum), float(weight_decay), ops.shape[0], _i32(ops), n,
            _f32(x) if x is not None else None, _i32(lab) if lab is not None else None,
            _f32(tgt) if tgt is not None else None, ctypes.byref(h)))
        self.h = h
        self.has_momentum = momentum != 0.0
        self._keep = (x, lab, tgt)
        self._opened = []
        return self

    def region(self) -> int:
        base, size = ctypes.c_void_p(), ctypes.c_size_t()
        N.check(self.lib.cdp_trainer_region(self.h, ctypes.byref(base), ctypes.byref(size)))
        return base.value

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        N.check(self.lib.cdp_trainer_ipc_handle(self.h, buf))
        return buf.raw

    def connect(self, regions):
        arr = (ctypes.c_void_p * len(regions))(*regions)
        N.check(self.lib.cdp_trainer_connect(self.h, arr))

    def connect_ipc(self, handles):
        """handles[r] = rank r's 64-byte IPC handle (own entry ignored)."""
        regions = []
        for r, hd in enumerate(handles):
            if r == self.rank:
                regions.append(self.region())
                continue
            ptr = ctypes.c_void_p()
            N.check(self.lib.cdp_ipc_open(ctypes.create_string_buffer(hd, 64), ctypes.byref(ptr)))
            self._opened.append(ptr.value)
            regions.append(ptr.value)
        self.connect(regions)

    def partial_tensor(self):
        """torch view (no copy) of the partial-sum buffer, for the NCCL all-reduce baseline."""
        import torch

        ptr, n = ctypes.c_void_p(), ctypes.c_size_t()
        N.check(self.lib.cdp_trainer_partial(self.h, ctypes.byref(ptr), ctypes.byref(n)))

        class _View:
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": "<f4", "data": (ptr.value, False),
                                        "version": 3}

        return torch.as_tensor(_View(), device="cuda")

    def apply_update(self):
        N.check(self.lib.cdp_trainer_apply_update(self.h))

    def ring_error(self) -> int:
        e = ctypes.c_int()
        N.check(self.lib.cdp_trainer_ring_error(self.h, ctypes.byref(e)))
        return e.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.cdp_trainer_destroy(self.h)
            self.h = None
        for p in getattr(self, "_opened", []):
            self.lib.cdp_ipc_close(ctypes.c_void_p(p))
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- params
    def set_params(self, flat: np.ndarray, which: int = -1):
        a = np.ascontiguousarray(flat, dtype=np.float32)
        assert a.size == self.P
        N.check(self.lib.cdp_trainer_set_params(self.h, which, _f32(a)))

    def get_params(self, which: int = 0) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        N.check(self.lib.cdp_trainer_get_params(self.h, which, _f32(out)))
        return out

    def set_velocity(self, flat: np.ndarray):
        a = np.ascontiguousarray(flat, dtype=np.float32)
        N.check(self.lib.cdp_trainer_set_velocity(self.h, _f32(a)))

    def get_velocity(self) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        N.check(self.lib.cdp_trainer_get_velocity(self.h, _f32(out)))
        return out

    def get_grad(self) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        N.check(self.lib.cdp_trainer_get_grad(self.h, _f32(out)))
        return out

    # -------------------------------------------------------------- steps
    def step(self, perm: np.ndarray, lr: float):
        p = np.ascontiguousarray(perm, dtype=np.int32)
        assert p.size == self.n_workers * self.micro_batch
        N.check(self.lib.cdp_trainer_step(self.h, _i32(p), float(lr)))

    def step_host_batch(self, x: np.ndarray, y: np.ndarray, lr: float):
        """Step whose inputs come from host memory (copied H2D inside the step)."""
        xa = np.ascontiguousarray(x, dtype=np.float32)
        if self.loss_kind == 1:
            ya = np.ascontiguousarray(y, dtype=np.int32)
            N.check(self.lib.cdp_trainer_step_host_batch(self.h, _f32(xa), _i32(ya), None, float(lr)))
        else:
            ya = np.ascontiguousarray(y, dtype=np.float32)
            N.check(self.lib.cdp_trainer_step_host_batch(self.h, _f32(xa), None, _f32(ya), float(lr)))
        self._keep_step = (xa, ya)

    def sync(self):
        N.check(self.lib.cdp_trainer_sync(self.h))

    def history(self, max_steps: int = 1 << 16):
        losses = np.empty(max_steps, dtype=np.float64)
        flags = np.empty((max_steps, 3), dtype=np.uint32)
        cnt = ctypes.c_int()
        N.check(self.lib.cdp_trainer_history(self.h, max_steps, losses.ctypes.data_as(N.c_double_p),
                                             flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                             ctypes.byref(cnt)))
        n = min(cnt.value, max_steps)
        return losses[:n].copy(), flags[:n].copy()

    def last(self):
        """(mean loss, flags[3]) of the most recent step; synchronises."""
        loss = ctypes.c_double()
        flags = (ctypes.c_uint32 * 3)()
        N.check(self.lib.cdp_trainer_last(self.h, ctypes.byref(loss), flags))
        return loss.value, tuple(flags)

    def step_host_batch_ptr(self, x_ptr: int, y_ptr: int, lr: float):
        """Host-batch step from raw (pinned) host pointers: x fp32, y int32 labels or fp32 targets."""
        if self.loss_kind == 1:
            N.check(self.lib.cdp_trainer_step_host_batch(self.h, ctypes.cast(x_ptr, N.c_float_p),
                                                         ctypes.cast(y_ptr, ctypes.POINTER(ctypes.c_int32)), None,
                                                         float(lr)))
        else:
            N.check(self.lib.cdp_trainer_step_host_batch(self.h, ctypes.cast(x_ptr, N.c_float_p), None,
                                                         ctypes.cast(y_ptr, N.c_float_p), float(lr)))

    def time_op(self, op: int, mask: int, iters: int) -> float:
        ms = ctypes.c_float()
        N.check(self.lib.cdp_trainer_time_op(self.h, op, mask, iters, ctypes.byref(ms)))
        return ms.value

    def mark(self, k: int):
        N.check(self.lib.cdp_trainer_mark(self.h, k))

    def elapsed(self, a: int, b: int) -> float:
        ms = ctypes.c_float()
        N.check(self.lib.cdp_trainer_elapsed(self.h, a, b, ctypes.byref(ms)))
        return ms.value

    def flush_l2(self):
        N.check(self.lib.cdp_trainer_flush_l2(self.h))

    def op_index(self, kind: int, worker: int, stage: int) -> int:
        rows = self.plan.ops if self.plan is not None else self.rank_ops
        for o, row in enumerate(rows):
            if row[0] == kind and row[1] == worker and row[2] == stage:
                return o
        raise KeyError((kind, worker, stage))

    def trace_step(self, perm: np.ndarray, lr: float, step: int) -> dict:
        """Run one step with %globaltimer stamps around every op; returns
        {(TaskKind, micro_batch, layer, step): (start_ns, end_ns)} (task end = max of both halves)."""
        from .schedule import TaskKind

        if not getattr(self, "_tracing", False):
            N.check(self.lib.cdp_trainer_set_trace(self.h, 1))
            self._tracing = True
        self.step(perm, lr)
        rows = self.plan.ops if self.plan is not None else self.rank_ops
        buf = np.zeros((len(rows), 4), dtype=np.uint64)
        N.check(self.lib.cdp_trainer_trace(self.h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(rows)))
        out = {}
        for o, row in enumerate(rows):
            kind = int(row[0])
            if kind == 2:
                continue
            s0, e0, s1, e1 = (int(v) for v in buf[o])
            out[(TaskKind.FORWARD if kind == 0 else TaskKind.BACKWARD, int(row[1]), int(row[2]), step)] = (
                s0, max(e0, e1))
        return out

    def stats(self) -> dict:
        out = np.zeros(6, dtype=np.int64)
        N.check(self.lib.cdp_trainer_stats(self.h, out.ctypes.data_as(N.c_int64_p), 6))
        return {"activation_bytes": int(out[0]), "param_state_bytes": int(out[1]), "kernels_per_step": int(out[2]),
                "next_step": int(out[3]), "streams": int(out[4]), "ops_per_step": int(out[5])}

    def stream_handle(self) -> int:
        s = ctypes.c_void_p()
        N.check(self.lib.cdp_trainer_stream(self.h, ctypes.byref(s)))
        return s.value or 0
