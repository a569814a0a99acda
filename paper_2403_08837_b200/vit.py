"""Vision Transformers on the device trainer (BASELINE configs[3]: ViT-B/16, 224x224).

The reference has no ViT; this is the north star's "layer compute of the named models"
for the CDP step (ViT GEMMs on tcgen05), parity-checked against a torch-CPU float64 restatement
(oracle/vit_torch.py, itself pinned to torchvision's VisionTransformer).  Conventions:

* torchvision `vit_b_16` structure: patch conv (kernel = stride = 16), class token, learned position
  embedding, 12 pre-LN blocks (LN eps 1e-6, fused qkv attention, 12 heads x 64, exact-erf GELU MLP
  3072), final LN, head on the class token; no dropout.
* Flat parameters, one hop unit per tensor (oracle/vit_torch.vit_specs): linear layers as
  [[W^T]; b] ([in + 1][out], the reference's [W][b] stage layout), LayerNorms [gamma | beta].
* bf16 operands / activations, fp32 residual stream, fp32 master state and momentum.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native as N
from .device import DTYPES

VIT_B16 = dict(image=224, patch=16, dim=768, depth=12, heads=12, mlp=3072, classes=1000)


def vit_units(image=224, patch=16, dim=768, depth=12, heads=12, mlp=3072, classes=1000):
    """[(name, shape, flops_per_sample)] per hop unit (fwd + bwd tensor-core flops of its GEMM)."""
    T = (image // patch) ** 2 + 1
    npch = T - 1
    out = [("patch", (patch * patch * 3 + 1, dim), 2 * 2 * npch * (patch * patch * 3 + 1) * dim),
           ("cls", (dim,), 0), ("pos", (T, dim), 0)]
    attn = 2 * 3 * 2 * T * T * dim  # scores + values, fwd and the two backward products each
    for i in range(depth):
        out += [(f"b{i}.ln1", (2 * dim,), 0),
                (f"b{i}.qkv", (dim + 1, 3 * dim), 6 * T * (dim + 1) * 3 * dim + attn),
                (f"b{i}.proj", (dim + 1, dim), 6 * T * (dim + 1) * dim),
                (f"b{i}.ln2", (2 * dim,), 0),
                (f"b{i}.fc1", (dim + 1, mlp), 6 * T * (dim + 1) * mlp),
                (f"b{i}.fc2", (mlp + 1, dim), 6 * T * (mlp + 1) * dim)]
    out += [("ln", (2 * dim,), 0), ("head", (dim + 1, classes), 6 * (dim + 1) * classes)]
    return out


def stage_partition(units, n_stages):
    """Contiguous groups of units with balanced FLOPs (vector units ride with their neighbours)."""
    flops = np.array([max(f, 1) for _, _, f in units], dtype=np.float64)
    cum = np.cumsum(flops)
    total = cum[-1]
    stage = np.empty(len(units), dtype=np.int32)
    s = 1
    for i in range(len(units)):
        while s < n_stages and cum[i] - flops[i] / 2 > total * s / n_stages:
            s += 1
        stage[i] = s
    for k in range(1, n_stages + 1):
        if not (stage == k).any():
            stage = np.repeat(np.arange(1, n_stages + 1), int(np.ceil(len(units) / n_stages)))[: len(units)]
            break
    return stage.astype(np.int32)


def vit_segments(units, depth):
    """Segment of every unit: 0 = embedding (patch, cls, pos), 1..depth = blocks, depth + 1 = final
    LN + head; and the per-segment tensor-core flops (the single-GPU executor's stage tasks run whole
    segments, so stage boundaries fall between segments)."""
    seg = np.array([0, 0, 0] + [1 + k // 6 for k in range(6 * depth)] + [depth + 1, depth + 1], dtype=np.int32)
    assert len(seg) == len(units)
    cost = np.zeros(depth + 2)
    for s, (_n, _shape, f) in zip(seg, units):
        cost[s] += f
    return seg, cost


def cyclic_plan(cfg, n_workers, rule=None):
    """Single-GPU CDP (rule) or DP (None) plan for `n_workers` micro-batches of this ViT on one GPU:
    (unit stage, SegmentPlan).  Segments are split into N FLOP-balanced contiguous stages; record
    pools: 0 = embedding records, 1 = block records (shared by all blocks), 2 = final records."""
    from .executor import compile_segment_plan, segment_partition

    units = vit_units(**cfg)
    depth = cfg["depth"]
    seg, cost = vit_segments(units, depth)
    seg_stage = segment_partition(np.maximum(cost, 1.0), n_workers)
    pool = [0] + [1] * depth + [2]
    return seg_stage[seg].astype(np.int32), compile_segment_plan(n_workers, seg_stage, pool, rule)


def vit_init(cfg, seed=0) -> np.ndarray:
    """Deterministic initialisation in the trainer layout (numpy PCG64): linear weights N(0, 0.02),
    biases 0, LayerNorm (1, 0), class token / position embedding N(0, 0.02)."""
    rng = np.random.default_rng([seed, 0xF0])
    parts = []
    for name, shape, _ in vit_units(**cfg):
        n = int(np.prod(shape))
        if name.endswith(("ln1", "ln2")) or name == "ln":
            c = shape[0] // 2
            parts.append(np.concatenate([np.ones(c), np.zeros(c)]))
        elif name in ("cls", "pos"):
            parts.append(rng.normal(0.0, 0.02, size=n))
        else:
            rows, cols = shape
            parts.append(np.concatenate([rng.normal(0.0, 0.02, size=(rows - 1, cols)), np.zeros((1, cols))]).ravel())
    return np.concatenate(parts)


def _i32p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


class DeviceVit:
    """One rank (worker) of CDP training of a ViT on this process's GPU.  dtype "bf16" (bf16 operands,
    fused attention) or "fp32" (3xTF32 operands, fp32 softmax: parity at fp32 tolerance)."""

    def __init__(self, cfg=None, micro_batch=32, world=1, rank=0, rule=None, momentum=0.0, weight_decay=0.0,
                 inputs=None, labels=None, stage_of_unit=None, trace=False, dtype="bf16"):
        if dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {sorted(DTYPES)}")
        self.dtype = dtype
        self.cfg = dict(VIT_B16 if cfg is None else cfg)
        self.lib = N.lib()
        self.micro_batch, self.world, self.rank = int(micro_batch), int(world), int(rank)
        self.units = vit_units(**self.cfg)
        self.stage = np.ascontiguousarray(stage_of_unit if stage_of_unit is not None
                                          else stage_partition(self.units, world), dtype=np.int32)
        fresh = np.ones(world, dtype=np.uint8)
        if rule is not None:
            if rule.n != world:
                raise ValueError("rule size must equal the number of ranks")
            rule.check_feasible()
            fresh = np.array([rule.reads_fresh(rank + 1, s) for s in range(1, world + 1)], dtype=np.uint8)
        x = lab = None
        n = 0
        if inputs is not None:
            x = np.ascontiguousarray(inputs, dtype=np.float32)
            lab = np.ascontiguousarray(labels, dtype=np.int32)
            n = x.shape[0]
        c = self.cfg
        h = ctypes.c_void_p()
        N.check(self.lib.cdp_vit_create_rank(
            c["image"], c["patch"], c["dim"], c["depth"], c["heads"], c["mlp"], c["classes"], self.micro_batch,
            world, rank, _i32p(self.stage), fresh.ctypes.data_as(N.c_u8_p), float(momentum), float(weight_decay), n,
            x.ctypes.data_as(N.c_float_p) if x is not None else None, _i32p(lab) if lab is not None else None,
            DTYPES[dtype], ctypes.byref(h)))
        self.h = h
        self._keep = (x, lab)
        if trace:
            N.check(self.lib.cdp_vit_set_trace(self.h, 1))
        np_, nu = ctypes.c_int64(), ctypes.c_int()
        # theta delivery along the reader order (see resnet.pull_chain); CDP_PULL_CHAIN=0: from the updater
        self.pull_chain = None
        if world > 1 and os.environ.get("CDP_PULL_CHAIN", "1") != "0":
            from .resnet import pull_chain

            self.pull_chain = pull_chain(rule, world, rank)
            N.check(self.lib.cdp_vit_pull_chain(self.h, _i32p(self.pull_chain), world))
        N.check(self.lib.cdp_vit_info(self.h, ctypes.byref(np_), ctypes.byref(nu)))
        assert nu.value == len(self.units), (nu.value, len(self.units))
        self.P = np_.value
        assert self.P == sum(int(np.prod(s)) for _, s, _ in self.units)
        self._opened = []

    @classmethod
    def single_gpu(cls, cfg=None, micro_batch=32, n_workers=4, rule=None, momentum=0.0, weight_decay=0.0,
                   inputs=None, labels=None, probe=True, trace=False, dtype="bf16"):
        """Single-GPU cyclic CDP (rule) or DP (rule None): `n_workers` micro-batches = stages on this
        GPU, stepped through the reference SINGLE_GPU_CDP / SINGLE_GPU_DP timeline with activation
        records from the plan's interval colouring (cdp_vit_create_cyclic).  step() takes
        n_workers * micro_batch indices, worker-major (ref models.py:173-185)."""
        self = cls.__new__(cls)
        if dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {sorted(DTYPES)}")
        self.dtype = dtype
        self.cfg = dict(VIT_B16 if cfg is None else cfg)
        self.lib = N.lib()
        self.micro_batch, self.world, self.rank = int(micro_batch), 1, 0
        self.n_workers = int(n_workers)
        self.units = vit_units(**self.cfg)
        stage, plan = cyclic_plan(self.cfg, self.n_workers, rule)
        self.stage, self.plan = np.ascontiguousarray(stage, dtype=np.int32), plan
        x = lab = None
        n = 0
        if inputs is not None:
            x = np.ascontiguousarray(inputs, dtype=np.float32)
            lab = np.ascontiguousarray(labels, dtype=np.int32)
            n = x.shape[0]
        c = self.cfg
        ops = np.ascontiguousarray(plan.ops, dtype=np.int32)
        slot = np.ascontiguousarray(plan.slot, dtype=np.int32)
        pools = np.ascontiguousarray(plan.pools, dtype=np.int32)
        fresh = np.ascontiguousarray(plan.fresh, dtype=np.uint8)
        h = ctypes.c_void_p()
        N.check(self.lib.cdp_vit_create_cyclic(
            c["image"], c["patch"], c["dim"], c["depth"], c["heads"], c["mlp"], c["classes"], self.micro_batch,
            self.n_workers, _i32p(self.stage), fresh.ctypes.data_as(N.c_u8_p), len(ops), _i32p(ops), _i32p(slot),
            _i32p(pools), float(momentum), float(weight_decay), int(bool(probe)), n,
            x.ctypes.data_as(N.c_float_p) if x is not None else None, _i32p(lab) if lab is not None else None,
            DTYPES[dtype], ctypes.byref(h)))
        self.h = h
        self._keep = (x, lab)
        if trace:
            N.check(self.lib.cdp_vit_set_trace(self.h, 1))
        np_, nu = ctypes.c_int64(), ctypes.c_int()
        N.check(self.lib.cdp_vit_info(self.h, ctypes.byref(np_), ctypes.byref(nu)))
        self.P = np_.value
        self._opened = []
        self.connect([self.region()])
        return self

    def region(self) -> int:
        b = ctypes.c_void_p()
        N.check(self.lib.cdp_vit_region(self.h, ctypes.byref(b)))
        return b.value

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        N.check(self.lib.cdp_vit_ipc_handle(self.h, buf))
        return buf.raw

    def connect(self, regions):
        N.check(self.lib.cdp_vit_connect(self.h, (ctypes.c_void_p * len(regions))(*regions)))

    def connect_ipc(self, handles):
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

    def set_params(self, flat, which=-1):
        a = np.ascontiguousarray(flat, dtype=np.float32)
        assert a.size == self.P
        N.check(self.lib.cdp_vit_set_params(self.h, which, a.ctypes.data_as(N.c_float_p)))

    def get_params(self, which=0) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        N.check(self.lib.cdp_vit_get_params(self.h, which, out.ctypes.data_as(N.c_float_p)))
        return out

    def step(self, perm, lr):
        p = np.ascontiguousarray(perm, dtype=np.int32)
        assert p.size == self.micro_batch * getattr(self, "n_workers", 1)
        N.check(self.lib.cdp_vit_step(self.h, _i32p(p), float(lr)))

    def step_host_batch_ptr(self, x_ptr: int, y_ptr: int, lr: float):
        N.check(self.lib.cdp_vit_step_host_batch(self.h, ctypes.cast(x_ptr, N.c_float_p),
                                                 ctypes.cast(y_ptr, ctypes.POINTER(ctypes.c_int)), float(lr)))

    def profile_step(self, perm, lr, serial=False, max_ops=4096):
        p = np.ascontiguousarray(perm, dtype=np.int32)
        NL = 48
        names = ctypes.create_string_buffer(max_ops * NL)
        fl, by = np.zeros(max_ops), np.zeros(max_ops)
        ms = np.zeros(max_ops, dtype=np.float32)
        n = ctypes.c_int()
        N.check(self.lib.cdp_vit_profile_step(self.h, _i32p(p), float(lr), int(serial), max_ops, names, NL,
                                              fl.ctypes.data_as(N.c_double_p), by.ctypes.data_as(N.c_double_p),
                                              ms.ctypes.data_as(N.c_float_p), ctypes.byref(n)))
        raw = names.raw
        return [(raw[i * NL:(i + 1) * NL].split(b"\0", 1)[0].decode(), float(fl[i]), float(by[i]), float(ms[i]))
                for i in range(min(n.value, max_ops))]

    def history(self, max_steps=1 << 14):
        losses = np.empty(max_steps)
        flags = np.empty((max_steps, 3), dtype=np.uint32)
        c = ctypes.c_int()
        N.check(self.lib.cdp_vit_history(self.h, max_steps, losses.ctypes.data_as(N.c_double_p),
                                         flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ctypes.byref(c)))
        k = min(c.value, max_steps)
        return losses[:k].copy(), flags[:k].copy()

    def sync(self):
        N.check(self.lib.cdp_vit_sync(self.h))

    def zero_drain(self):
        pass

    def access_trace(self, max_records=1 << 16):
        """Executed-version records since the last call (trace=True trainers; _native.read_access_trace)."""
        return N.read_access_trace(self.lib.cdp_vit_trace, self.h, max_records)

    def ring_error(self) -> int:
        e = ctypes.c_int()
        N.check(self.lib.cdp_vit_ring_error(self.h, ctypes.byref(e)))
        return e.value

    def stats(self) -> dict:
        out = np.zeros(11, dtype=np.int64)
        N.check(self.lib.cdp_vit_stats(self.h, out.ctypes.data_as(N.c_int64_p), 11))
        return {"activation_bytes": int(out[0]), "param_state_bytes": int(out[1]), "kernels_per_step": int(out[2]),
                "tensor_flops_per_step": int(out[3]), "live_record_high_water_bytes": int(out[4]),
                "record_bytes": [int(v) for v in out[5:8]], "record_slots": [int(v) for v in out[8:11]]}

    def mark(self, k):
        N.check(self.lib.cdp_vit_mark(self.h, k))

    def elapsed(self, a, b) -> float:
        ms = ctypes.c_float()
        N.check(self.lib.cdp_vit_elapsed(self.h, a, b, ctypes.byref(ms)))
        return ms.value

    def flush_l2(self):
        N.check(self.lib.cdp_vit_flush_l2(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.cdp_vit_destroy(self.h)
            self.h = None
        for p in getattr(self, "_opened", []):
            self.lib.cdp_ipc_close(ctypes.c_void_p(p))
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
