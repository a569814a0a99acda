"""ResNets on the device trainer (BASELINE configs[1]: ResNet-18, CIFAR-10 shape; configs[2,4]: ResNet-50,
ImageNet shape).

The reference has no ResNet; this is the north star's "layer
compute of the named models" for the CDP step, parity-checked against a
torch-CPU restatement of the same step (oracle/resnet_torch.py, "parity
unpinned" by the reference).  Conventions:

* ResNet-18 CIFAR variant (`PAPER.md:312`): 3x3 stride-1 stem, no max-pool,
  stages of BasicBlocks (widths 64/128/256/512, depths 2/2/2/2), 1x1
  projection shortcuts, global average pool, linear classifier.
* ResNet-50 (torchvision v1.5 layout): 7x7/s2 stem + 3x3/s2 max pool,
  Bottleneck blocks (1x1, 3x3 with the stride, 1x1 x4), depths 3/4/6/3.
* Batch norm in training mode with per-micro-batch statistics; running
  statistics are not tracked (SURVEY §7 hard part 4 — one convention fixed).
* Parameter tensors in torchvision `named_parameters` order; flat layout per
  tensor: conv `[R][S][Cin][Cout]`, BN `[gamma | beta]`, fc `[[W^T]; b]`.
* Stages: contiguous tensor groups, FLOP-balanced (`stage_partition`).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native as N
from .device import DTYPES

RESNET18 = dict(widths=(64, 128, 256, 512), depths=(2, 2, 2, 2), block="basic", stem="cifar")
RESNET50 = dict(widths=(64, 128, 256, 512), depths=(3, 4, 6, 3), block="bottleneck", stem="imagenet")
BLOCKS = {"basic": 0, "bottleneck": 1}
STEMS = {"cifar": 0, "imagenet": 1}


def layer_specs(widths, depths, in_ch=3, hw=32, block="basic", stem="cifar", classes=10):
    """[(kind, shape, flops_per_sample)] per parameter tensor, in the trainer's (torchvision) order.

    flops = forward + backward (data and weight gradients) tensor-core flops of the conv."""
    out = []

    def conv(cin, cout, r, stride, H, pad=None):
        pad = r // 2 if pad is None else pad
        Ho = (H + 2 * pad - r) // stride + 1
        out.append(("conv", (r, r, cin, cout), 2 * 3 * r * r * cin * cout * Ho * Ho))
        out.append(("bn", (2 * cout,), 0))
        return Ho

    H = hw
    if stem == "cifar":
        H = conv(in_ch, widths[0], 3, 1, H)
    else:
        H = conv(in_ch, widths[0], 7, 2, H, pad=3)
        H = (H + 2 - 3) // 2 + 1
    cin = widths[0]
    exp = 4 if block == "bottleneck" else 1
    for l, (w, d) in enumerate(zip(widths, depths)):
        for k in range(d):
            stride = 2 if (l > 0 and k == 0) else 1
            if block == "basic":
                Ho = conv(cin, w, 3, stride, H)
                conv(w, w, 3, 1, Ho)
            else:
                conv(cin, w, 1, 1, H)
                Ho = conv(w, w, 3, stride, H)
                conv(w, w * exp, 1, 1, Ho)
            if stride != 1 or cin != w * exp:
                conv(cin, w * exp, 1, stride, H)
            cin, H = w * exp, Ho
    out.append(("fc", (cin + 1, classes), 2 * 3 * cin * classes))
    return out


def block_starts(widths, depths, block="basic", stem="cifar"):
    """Tensor indices (layer_specs order) where a residual block, or the classifier, starts."""
    starts, i, cin = [], 2, widths[0]
    exp = 4 if block == "bottleneck" else 1
    for l, (w, d) in enumerate(zip(widths, depths)):
        for k in range(d):
            stride = 2 if (l > 0 and k == 0) else 1
            starts.append(i)
            i += 2 * (2 if block == "basic" else 3) + (2 if (stride != 1 or cin != w * exp) else 0)
            cin = w * exp
    starts.append(i)  # the classifier
    return starts


def zero_partition(widths, depths, hw, block, stem, classes, n_stages):
    """ZeRO-CDP stages: balanced parameter counts with boundaries only at residual-block (or classifier)
    starts.  A block's last BN and its projection shortcut are one BN-backward kernel and its output's
    BN apply reads both, so a boundary inside a block would interleave two stages' use windows on a rank,
    against the reference order the state-frame reuse waits rely on (csrc/resnet_trainer.cu)."""
    specs = layer_specs(widths, depths, 3, hw, block, stem, classes)
    return stage_partition(specs, n_stages, "params", starts=block_starts(widths, depths, block, stem))


def stage_partition(specs, n_stages, by="flops", starts=None):
    """Contiguous groups of tensors with balanced FLOPs (BN/fc ride with their neighbour), or balanced
    parameter counts (by="params"); `starts`: the only tensor indices a stage may begin at (besides 0)."""
    if starts is not None:
        w = np.array([max(float(np.prod(s)), 1.0) if by == "params" else max(f, 1) for _, s, f in specs])
        cum = np.concatenate([[0.0], np.cumsum(w)])
        cand = sorted(set(int(c) for c in starts if 0 < c < len(specs)))
        if len(cand) < n_stages - 1:
            raise ValueError(f"{n_stages} stages need {n_stages - 1} block boundaries, the model has {len(cand)}")
        bounds, lo = [], 0
        for k in range(1, n_stages):
            # the remaining boundaries must still fit after this one
            options = [c for c in cand if c > lo and len([x for x in cand if x > c]) >= n_stages - 1 - k]
            c = min(options, key=lambda c: abs(cum[c] - cum[-1] * k / n_stages))
            bounds.append(c)
            lo = c
        stage = np.ones(len(specs), dtype=np.int32)
        for b in bounds:
            stage[b:] += 1
        return stage
    if by == "params":
        flops = np.array([max(float(np.prod(s)), 1.0) for _, s, _ in specs], dtype=np.float64)
    else:
        flops = np.array([max(f, 1) for _, _, f in specs], dtype=np.float64)
    cum = np.cumsum(flops)
    total = cum[-1]
    stage = np.empty(len(specs), dtype=np.int32)
    s = 1
    for i in range(len(specs)):
        while s < n_stages and cum[i] - flops[i] / 2 > total * s / n_stages:
            s += 1
        stage[i] = s
    # every stage non-empty and contiguous
    for k in range(1, n_stages + 1):
        if not (stage == k).any():
            stage = np.repeat(np.arange(1, n_stages + 1), int(np.ceil(len(specs) / n_stages)))[: len(specs)]
            break
    return stage.astype(np.int32)


# ----------------------------------------------------------------------------- layout conversion
def torch_to_flat(model) -> np.ndarray:
    """torch ResNet (oracle/resnet_torch.TorchResNet) -> flat float64 theta in the trainer layout."""
    parts = []
    for name, p in _ordered(model):
        a = p.detach().double().cpu().numpy()
        if name.endswith("conv"):
            parts.append(np.transpose(a, (2, 3, 1, 0)).ravel())  # [Cout][Cin][R][S] -> [R][S][Cin][Cout]
        elif name.endswith("bn"):
            parts.append(np.concatenate([a[0], a[1]]))
        else:  # fc: (weight [classes][C], bias [classes]) -> [[W^T]; b]
            parts.append(np.concatenate([a[0].T, a[1][None, :]]).ravel())
    return np.concatenate(parts)


def flat_to_tensors(flat: np.ndarray, specs) -> list:
    out, pos = [], 0
    for kind, shape, _ in specs:
        n = int(np.prod(shape))
        out.append(flat[pos:pos + n])
        pos += n
    return out


def _ordered(model):
    """(name, tensor-or-pair) in trainer order, from an oracle torch model (oracle/resnet_torch.TorchResNet)."""
    items = [("stem.conv", model.stem_conv.weight), ("stem.bn", (model.stem_bn.weight, model.stem_bn.bias))]
    for bi, b in enumerate(model.blocks):
        for ci, (cv, bn) in enumerate(zip(b.convs, b.bns)):
            items.append((f"b{bi}.c{ci}.conv", cv.weight))
            items.append((f"b{bi}.c{ci}.bn", (bn.weight, bn.bias)))
        if b.ds_conv is not None:
            items.append((f"b{bi}.ds.conv", b.ds_conv.weight))
            items.append((f"b{bi}.ds.bn", (b.ds_bn.weight, b.ds_bn.bias)))
    items.append(("fc", (model.fc.weight, model.fc.bias)))
    out = []
    for name, p in items:
        if isinstance(p, tuple):
            out.append((name, _Pair(p)))
        else:
            out.append((name, p))
    return out


class _Pair:
    def __init__(self, pair):
        self.pair = pair

    def detach(self):
        return self

    def double(self):
        return self

    def cpu(self):
        return self

    def numpy(self):
        return [t.detach().double().cpu().numpy() for t in self.pair]


# ----------------------------------------------------------------------------- device trainer
def _i32p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


class DeviceResNet:
    """One rank (worker) of CDP training of a ResNet (BasicBlock / Bottleneck, CIFAR / ImageNet stem)
    on this process's GPU."""

    def __init__(self, widths=RESNET18["widths"], depths=RESNET18["depths"], micro_batch=128, world=1, rank=0,
                 rule=None, dtype="bf16", momentum=0.0, weight_decay=0.0, inputs=None, labels=None, classes=10,
                 image_hw=32, stage_of_tensor=None, block="basic", stem="cifar", zero=False, dp_allreduce=False,
                 trace=False, zero_frames=True):
        self.lib = N.lib()
        self.widths, self.depths = tuple(widths), tuple(depths)
        self.block, self.stem, self.classes, self.image_hw = block, stem, int(classes), int(image_hw)
        self.micro_batch, self.world, self.rank = int(micro_batch), int(world), int(rank)
        self.dtype = dtype
        self.specs = layer_specs(self.widths, self.depths, 3, image_hw, block, stem, classes)
        n_t = len(self.specs)
        self.stage = np.ascontiguousarray(stage_of_tensor if stage_of_tensor is not None
                                          else zero_partition(self.widths, self.depths, image_hw, block, stem,
                                                              classes, world) if (zero and zero_frames and world > 1)
                                          else stage_partition(self.specs, world),
                                          dtype=np.int32)
        fresh = np.ones(world, dtype=np.uint8)
        if rule is not None:
            if rule.n != world:
                raise ValueError("rule size must equal the number of ranks")
            rule.check_feasible()
            fresh = np.array([rule.reads_fresh(rank + 1, s) for s in range(1, world + 1)], dtype=np.uint8)
        self.fresh = fresh
        w = np.asarray(self.widths, dtype=np.int32)
        d = np.asarray(self.depths, dtype=np.int32)
        x = lab = None
        n = 0
        if inputs is not None:
            x = np.ascontiguousarray(inputs, dtype=np.float32)
            lab = np.ascontiguousarray(labels, dtype=np.int32)
            n = x.shape[0]
        self.zero = bool(zero) and world > 1
        ztab = None
        if self.zero:
            from .zero import zero_plan

            if rule is None or any(rule.reads_fresh(i, j) != (j >= world - i + 1)
                                   for i in range(1, world + 1) for j in range(1, world + 1)):
                raise ValueError("ZeRO-CDP uses the CDP-v2 placement (ref schedule.py:471): rule must be cdp-v2")
            ztab = zero_plan(world).table()
        self._ztab = ztab
        h = ctypes.c_void_p()
        N.check(self.lib.cdp_resnet_create_rank(
            len(w), _i32p(w), _i32p(d), BLOCKS[block], STEMS[stem], 3, image_hw, image_hw, classes, self.micro_batch, world, rank,
            _i32p(self.stage), fresh.ctypes.data_as(N.c_u8_p), DTYPES[dtype], float(momentum), float(weight_decay),
            n, x.ctypes.data_as(N.c_float_p) if x is not None else None, _i32p(lab) if lab is not None else None,
            _i32p(ztab) if ztab is not None else None,
            (1 if dp_allreduce else 0) | (2 if trace else 0) | (0 if zero_frames else 4),
            ctypes.byref(h)))
        self.dp_allreduce = bool(dp_allreduce)
        # ZeRO-CDP keeps two stage frames of parameter state per rank (include/cdp_b200.h); full replicas
        # with zero_frames=False
        self.zero_frames = self.zero and bool(zero_frames)
        # theta delivery along the reader order (csrc/rank_common.cuh chain kernels); CDP_PULL_CHAIN=0: every
        # reader pulls from the updater
        self.pull_chain = None
        if world > 1 and not self.zero and not dp_allreduce and os.environ.get("CDP_PULL_CHAIN", "1") != "0":
            self.pull_chain = pull_chain(rule, world, rank)
            N.check(self.lib.cdp_resnet_pull_chain(h, _i32p(self.pull_chain), world))
        if self.zero_frames:
            from .zero import frame_drain_plan

            rows = np.ascontiguousarray(np.array(frame_drain_plan(world)[rank], dtype=np.int32).reshape(-1, 5))
            N.check(self.lib.cdp_resnet_zero_drain_plan(h, _i32p(rows) if len(rows) else None, len(rows)))
        self.h = h
        self._keep = (x, lab)
        np_, nt = ctypes.c_int64(), ctypes.c_int()
        N.check(self.lib.cdp_resnet_info(self.h, ctypes.byref(np_), ctypes.byref(nt), None, None))
        assert nt.value == n_t, (nt.value, n_t)
        self.P = np_.value
        self._opened = []

    def region(self) -> int:
        b = ctypes.c_void_p()
        N.check(self.lib.cdp_resnet_region(self.h, ctypes.byref(b)))
        return b.value

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        N.check(self.lib.cdp_resnet_ipc_handle(self.h, buf))
        return buf.raw

    def connect(self, regions):
        N.check(self.lib.cdp_resnet_connect(self.h, (ctypes.c_void_p * len(regions))(*regions)))

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
        N.check(self.lib.cdp_resnet_set_params(self.h, which, a.ctypes.data_as(N.c_float_p)))

    def get_params(self, which=0) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        N.check(self.lib.cdp_resnet_get_params(self.h, which, out.ctypes.data_as(N.c_float_p)))
        return out

    def step(self, perm, lr):
        p = np.ascontiguousarray(perm, dtype=np.int32)
        assert p.size == self.micro_batch
        N.check(self.lib.cdp_resnet_step(self.h, _i32p(p), float(lr)))

    def step_host_batch_ptr(self, x_ptr: int, y_ptr: int, lr: float):
        """End-to-end step from raw (pinned) host pointers: x fp32 NHWC [B][H][W][3], y int32 labels."""
        N.check(self.lib.cdp_resnet_step_host_batch(self.h, ctypes.cast(x_ptr, N.c_float_p),
                                                    ctypes.cast(y_ptr, ctypes.POINTER(ctypes.c_int)), float(lr)))

    def step_host_batch_async(self, x_ptr: int, y_ptr: int, lr: float, slot: int):
        """Pipelined step on a pinned host batch (include/cdp_b200.h): its H2D copy overlaps the previous
        step; do not rewrite the host buffers before a sync."""
        N.check(self.lib.cdp_resnet_step_host_batch_async(self.h, ctypes.cast(x_ptr, N.c_float_p),
                                                          ctypes.cast(y_ptr, N.c_int_p), float(lr), int(slot)))

    def step_host_batch(self, x, y, lr):
        xa = np.ascontiguousarray(x, dtype=np.float32)
        ya = np.ascontiguousarray(y, dtype=np.int32)
        assert xa.shape[0] == self.micro_batch and ya.shape[0] == self.micro_batch
        self.step_host_batch_ptr(xa.ctypes.data, ya.ctypes.data, lr)
        self._keep_step = (xa, ya)

    def last_loss(self) -> float:
        out = ctypes.c_double()
        N.check(self.lib.cdp_resnet_last_loss(self.h, ctypes.byref(out)))
        return out.value

    def profile_step(self, perm, lr, serial=False, max_ops=4096):
        """One real training step, launched eagerly with CUDA events around every kernel (on the stream it is
        launched on; serial=True puts every launch on one stream so durations are not inflated by the
        concurrent stream).  Returns [(name, flops, bytes, ms)] in launch order."""
        p = np.ascontiguousarray(perm, dtype=np.int32)
        NL = 48
        names = ctypes.create_string_buffer(max_ops * NL)
        fl = np.zeros(max_ops)
        by = np.zeros(max_ops)
        ms = np.zeros(max_ops, dtype=np.float32)
        n = ctypes.c_int()
        N.check(self.lib.cdp_resnet_profile_step(self.h, _i32p(p), float(lr), int(serial), max_ops, names, NL,
                                                 fl.ctypes.data_as(N.c_double_p), by.ctypes.data_as(N.c_double_p),
                                                 ms.ctypes.data_as(N.c_float_p), ctypes.byref(n)))
        k = min(n.value, max_ops)
        raw = names.raw
        return [(raw[i * NL:(i + 1) * NL].split(b"\0", 1)[0].decode(), float(fl[i]), float(by[i]), float(ms[i]))
                for i in range(k)]

    def history(self, max_steps=1 << 14):
        losses = np.empty(max_steps)
        flags = np.empty((max_steps, 3), dtype=np.uint32)
        c = ctypes.c_int()
        N.check(self.lib.cdp_resnet_history(self.h, max_steps, losses.ctypes.data_as(N.c_double_p),
                                            flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ctypes.byref(c)))
        n = min(c.value, max_steps)
        return losses[:n].copy(), flags[:n].copy()

    # ---- DP all-reduce baseline (ref comm.py:70-90)
    def partial_tensor(self):
        """torch view (no copy) of the flat gradient buffer, summed across ranks by the caller."""
        import torch

        ptr, n = ctypes.c_void_p(), ctypes.c_size_t()
        N.check(self.lib.cdp_resnet_partial(self.h, ctypes.byref(ptr), ctypes.byref(n)))

        class _View:
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": "<f4", "data": (ptr.value, False),
                                        "version": 3}

        return torch.as_tensor(_View(), device="cuda")

    def stream_handle(self) -> int:
        s = ctypes.c_void_p()
        N.check(self.lib.cdp_resnet_stream(self.h, ctypes.byref(s)))
        return s.value or 0

    def apply_update(self, first_tensor=0, end_tensor=None):
        """Update from the summed flat gradient; a tensor range updates only those tensors (ZeRO-DP)."""
        if first_tensor == 0 and end_tensor is None:
            N.check(self.lib.cdp_resnet_apply_update(self.h))
        else:
            end = len(self.specs) if end_tensor is None else int(end_tensor)
            N.check(self.lib.cdp_resnet_apply_update_range(self.h, int(first_tensor), end))

    def theta_tensor(self, which=0):
        """torch view (no copy) of theta slot `which` (0: the version the next step reads fresh)."""
        import torch

        ptr, nb, ld = ctypes.c_void_p(), ctypes.c_size_t(), ctypes.c_int()
        N.check(self.lib.cdp_resnet_buffer(self.h, b"theta", int(which), ctypes.byref(ptr), ctypes.byref(nb),
                                           ctypes.byref(ld)))

        class _View:
            __cuda_array_interface__ = {"shape": (nb.value // 4,), "typestr": "<f4", "data": (ptr.value, False),
                                        "version": 3}

        return torch.as_tensor(_View(), device="cuda")

    def pack_range(self, which, first_tensor, end_tensor):
        """Repack the GEMM copies of tensors [first, end) after theta slot `which` was written externally."""
        N.check(self.lib.cdp_resnet_pack_range(self.h, int(which), int(first_tensor), int(end_tensor)))

    def tensor_bases(self) -> np.ndarray:
        np_, nt = ctypes.c_int64(), ctypes.c_int()
        N.check(self.lib.cdp_resnet_info(self.h, ctypes.byref(np_), ctypes.byref(nt), None, None))
        base = np.zeros(nt.value, dtype=np.int64)
        N.check(self.lib.cdp_resnet_info(self.h, ctypes.byref(np_), ctypes.byref(nt),
                                         base.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), None))
        return base

    def zero_state(self, which=0):
        """ZeRO-CDP frames: (this rank's frame contents in the full layout, last finished use per tensor)."""
        n_t = len(self.specs)
        theta = np.zeros(self.P, dtype=np.float32)
        last = np.zeros(n_t, dtype=np.uint32)
        N.check(self.lib.cdp_resnet_zero_state(self.h, int(which), theta.ctypes.data_as(N.c_float_p),
                                               last.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
        return theta, last

    def zero_drain(self):
        """ZeRO-CDP: publish the next step's forward uses (call on every rank before synchronising at the
        end of a run; see include/cdp_b200.h)."""
        if self.zero:
            N.check(self.lib.cdp_resnet_zero_drain(self.h))

    def sync(self):
        N.check(self.lib.cdp_resnet_sync(self.h))

    def ring_error(self) -> int:
        e = ctypes.c_int()
        N.check(self.lib.cdp_resnet_ring_error(self.h, ctypes.byref(e)))
        return e.value

    def stats(self) -> dict:
        out = np.zeros(6, dtype=np.int64)
        N.check(self.lib.cdp_resnet_stats(self.h, out.ctypes.data_as(N.c_int64_p), 6))
        return {"activation_bytes": int(out[0]), "param_state_bytes": int(out[1]), "kernels_per_step": int(out[2]),
                "tensor_flops_per_step": int(out[3]), "gradient_scratch_bytes": int(out[4]),
                "zero_state_bytes_per_step": int(out[5])}

    def mark(self, k):
        N.check(self.lib.cdp_resnet_mark(self.h, k))

    def elapsed(self, a, b) -> float:
        ms = ctypes.c_float()
        N.check(self.lib.cdp_resnet_elapsed(self.h, a, b, ctypes.byref(ms)))
        return ms.value

    def buffer(self, name, index=0, dtype=np.float32, rows=None):
        """Host copy of one internal device buffer (tests / diagnostics; include/cdp_b200.h
        cdp_resnet_buffer).  With `rows`, a [rows][ld] view."""
        ptr, nb, ld = ctypes.c_void_p(), ctypes.c_size_t(), ctypes.c_int()
        N.check(self.lib.cdp_resnet_buffer(self.h, name.encode(), int(index), ctypes.byref(ptr), ctypes.byref(nb),
                                           ctypes.byref(ld)))
        self.sync()
        out = np.empty(nb.value // np.dtype(dtype).itemsize, dtype=dtype)
        N.memcpy_d2h(out.ctypes.data, ptr.value, out.nbytes)
        if rows is not None:
            out = out[: rows * ld.value].reshape(rows, ld.value)
        return out

    def access_trace(self, max_records=1 << 16):
        """Executed-version records since the last call (trace=True trainers; _native.read_access_trace)."""
        return N.read_access_trace(self.lib.cdp_resnet_trace, self.h, max_records)

    def activation_shapes(self):
        """[(role, H, W, C)] of the trainer's activation buffers in creation order: "relu" (a ReLU output:
        stem, block inner and block output activations) or "pool" (the ImageNet stem's max-pool output)."""
        out = []
        H = self.image_hw
        w0 = self.widths[0]
        if self.stem == "cifar":
            out.append(("relu", H, H, w0))
        else:
            H = (H + 6 - 7) // 2 + 1
            out.append(("relu", H, H, w0))
            H = (H + 2 - 3) // 2 + 1
            out.append(("pool", H, H, w0))
        cin = w0
        exp = 4 if self.block == "bottleneck" else 1
        for l, (w, d) in enumerate(zip(self.widths, self.depths)):
            for k in range(d):
                stride = 2 if (l > 0 and k == 0) else 1
                Ho = (H - 1) // stride + 1
                if self.block == "basic":
                    out += [("relu", Ho, Ho, w), ("relu", Ho, Ho, w)]
                else:
                    out += [("relu", H, H, w), ("relu", Ho, Ho, w), ("relu", Ho, Ho, w * exp)]
                cin, H = w * exp, Ho
        return out

    def branch_decisions(self):
        """The last step's ReLU masks (activation > 0, NCHW bool, forward order) and max-pool window argmaxes
        ([B, C, Ho, Wo], or None), read from the device: the kink decisions a float64 restatement needs to
        follow the same branch where its own value is within rounding of a switching point."""
        B = self.micro_batch
        relu, pool = [], None
        fp32 = self.dtype == "fp32"
        for a, (role, H, W, C) in enumerate(self.activation_shapes()):
            rows = B * H * W
            if fp32:
                v = self.buffer("act_hi", a, np.float32, rows)[:, :C].astype(np.float64) + \
                    self.buffer("act_lo", a, np.float32, rows)[:, :C]
            else:
                raw = self.buffer("act_hi", a, np.uint16, rows)[:, :C].astype(np.uint32) << 16
                v = raw.view(np.float32)
            if role == "relu":
                relu.append(np.ascontiguousarray((v > 0).reshape(B, H, W, C).transpose(0, 3, 1, 2)))
            else:
                arg = self.buffer("pool_arg", 0, np.uint8)[: rows * C].reshape(B, H, W, C)
                pool = np.ascontiguousarray(arg.transpose(0, 3, 1, 2).astype(np.int64))
        return relu, pool

    def flush_l2(self):
        N.check(self.lib.cdp_resnet_flush_l2(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.cdp_resnet_destroy(self.h)
            self.h = None
        for p in getattr(self, "_opened", []):
            self.lib.cdp_ipc_close(ctypes.c_void_p(p))
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_params(specs, seed=0) -> np.ndarray:
    """Deterministic initialisation in the trainer layout (numpy PCG64): conv He-normal (fan_in = R*S*Cin),
    BN gamma = 1 / beta = 0, classifier U(-1/sqrt(C), 1/sqrt(C)) for W and b (torch's Linear bounds)."""
    rng = np.random.default_rng([seed, 0xE0])
    parts = []
    for kind, shape, _ in specs:
        if kind == "conv":
            r, s, cin, cout = shape
            parts.append(rng.normal(0.0, np.sqrt(2.0 / (r * s * cin)), size=r * s * cin * cout))
        elif kind == "bn":
            c = shape[0] // 2
            parts.append(np.concatenate([np.ones(c), np.zeros(c)]))
        else:
            rows, classes = shape
            b = 1.0 / np.sqrt(rows - 1)
            parts.append(rng.uniform(-b, b, size=rows * classes))
    return np.concatenate(parts)


def synthetic_images(n, seed=0, hw=32, classes=10):
    """x ~ N(0,1) NHWC [n][hw][hw][3] float32, labels uniform in [0, classes) from default_rng([seed, 0xD0])."""
    return synthetic_cifar(n, seed, hw, classes)


def synthetic_cifar(n, seed=0, hw=32, classes=10):
    """x ~ N(0,1) NHWC [n][hw][hw][3], labels uniform in [0, classes) from default_rng([seed, 0xD0])."""
    rng = np.random.default_rng([seed, 0xD0])
    return rng.normal(0.0, 1.0, size=(n, hw, hw, 3)).astype(np.float32), rng.integers(0, classes, size=n).astype(np.int32)


class ZeroDpRank:
    """ZeRO-DP baseline rank (ref comm.py:108-124, costs.py:140-153): stage s is owned by rank s - 1;
    before the step every owner broadcasts its stage's current parameters (NCCL / gloo broadcast on
    the trainer stream, the non-owners repack their GEMM copies), the step computes this rank's
    gradient (the DP all-reduce trainer's gradient-only epilogues), the gradient of every stage is
    reduced to its owner and only the owner updates that stage.  The reference moves 2 Psi_P per
    device per step (a broadcast for the forward and one for the backward of each stage, its states
    freed in between); this realisation keeps the broadcast parameters resident across the step, so
    it moves Psi_P of parameters (broadcast) + Psi_P of gradients (reduce) — `bytes_per_step` reports
    what it moves.  Not the hot path: the comparison point for ZeRO-CDP's P2P state passing."""

    def __init__(self, trainer: "DeviceResNet", group=None):
        import torch
        import torch.distributed as dist

        if not trainer.dp_allreduce:
            raise ValueError("ZeRO-DP runs on a DP all-reduce (gradient-only) trainer")
        self.tr, self.group = trainer, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        base = trainer.tensor_bases()
        n_t = len(trainer.specs)
        ends = list(base[1:]) + [trainer.P]
        self.ranges = []  # per stage: (first tensor, end tensor, first param, end param)
        for s in range(1, self.world + 1):
            idx = [k for k in range(n_t) if int(trainer.stage[k]) == s]
            if not idx or idx != list(range(idx[0], idx[-1] + 1)):
                raise ValueError("stages must be contiguous tensor ranges")
            self.ranges.append((idx[0], idx[-1] + 1, int(base[idx[0]]), int(ends[idx[-1]])))
        h = trainer.stream_handle()
        self.ext = torch.cuda.ExternalStream(h) if h else None  # None: host tensors (CPU tests)
        self.gloo = dist.get_backend(group) == "gloo"
        self.grad = trainer.partial_tensor()
        other = sum(r[3] - r[2] for i, r in enumerate(self.ranges) if i != self.rank)
        # this rank's traffic per step: the parameters of the stages it does not own (received by
        # broadcast) and its gradient of those stages (sent to their owners by the reduce)
        self.bytes_per_step = 8 * other

    def broadcast(self):
        import torch.distributed as dist

        theta = self.tr.theta_tensor(0)
        with self._on_stream():
            for s, (t0, t1, p0, p1) in enumerate(self.ranges):
                dist.broadcast(theta[p0:p1], src=s, group=self.group)
        for s, (t0, t1, p0, p1) in enumerate(self.ranges):
            if s != self.rank:
                self.tr.pack_range(0, t0, t1)

    def reduce_update(self):
        import torch.distributed as dist

        with self._on_stream():
            for s, (t0, t1, p0, p1) in enumerate(self.ranges):
                if self.gloo:  # gloo has no CUDA reduce: the all-reduce gives the owner the same sum
                    dist.all_reduce(self.grad[p0:p1], group=self.group)
                else:
                    dist.reduce(self.grad[p0:p1], dst=s, group=self.group)
        t0, t1, _, _ = self.ranges[self.rank]
        self.tr.apply_update(t0, t1)

    def _on_stream(self):
        import contextlib

        import torch

        return torch.cuda.stream(self.ext) if self.ext is not None else contextlib.nullcontext()

    def step(self, perm, lr):
        self.broadcast()
        self.tr.step(perm, lr)
        self.reduce_update()


def pull_chain(rule, world: int, rank: int) -> np.ndarray:
    """[world stages][2] (predecessor, successor) of `rank` in the order the readers (ranks 0 .. world-2; the
    last rank updates) read each new version of a stage: fresh readers at step v in worker order, then stale
    readers at step v + 1 (ref rules.py:45-51); -1: the updater / none."""
    out = np.full((world, 2), -1, dtype=np.int32)
    readers = range(world - 1)
    for j in range(1, world + 1):
        fresh = [rule is None or rule.reads_fresh(r + 1, j) for r in readers]
        order = [r for r in readers if fresh[r]] + [r for r in readers if not fresh[r]]
        if rank in order:
            k = order.index(rank)
            out[j - 1, 0] = order[k - 1] if k > 0 else -1
            out[j - 1, 1] = order[k + 1] if k + 1 < len(order) else -1
    return out


def gather_zero_params(ranks, which=0) -> np.ndarray:
    """The newest parameter state of a ZeRO-CDP (frames) job: every tensor from the rank whose last finished
    use of it is the latest (call after zero_drain + sync on every rank).  Full-replica ranks: the last
    rank's copy (the updater holds every stage's newest version)."""
    if not ranks[0].zero_frames:
        return ranks[-1].get_params(which)
    states = [r.zero_state(which) for r in ranks]
    base = [int(b) for b in ranks[0].tensor_bases()] + [ranks[0].P]
    out = np.zeros(ranks[0].P, dtype=np.float32)
    for i in range(len(base) - 1):
        holder = max(range(len(ranks)), key=lambda r: int(states[r][1][i]))
        out[base[i]:base[i + 1]] = states[holder][0][base[i]:base[i + 1]]
    return out
