"""ORACLE — TEST INFRASTRUCTURE ONLY.  torch-CPU restatement of the CDP step on
ResNets (BasicBlock / Bottleneck, CIFAR / ImageNet stem; BASELINE configs[1..2,4]); the reference has no ResNet, so this
restatement is "parity unpinned" by the reference: the reference's
`_advance` semantics (oracle/engine.advance: per-(micro-batch, stage) version
choice, ascending accumulation, SGD-momentum update) applied to per-micro-batch
gradients computed here with torch autograd in float64.

Model conventions are those of paper_2403_08837_b200/resnet.py (CIFAR stem,
training-mode batch norm with per-micro-batch statistics, eps 1e-5).

Kinks.  ReLU and max pool are not differentiable at their switching points: a
pre-activation within fp32 rounding of 0 (or two max-pool window entries within
rounding of each other) can take a different branch in the fp32 device step and
in this float64 step, and one such flip moves every upstream gradient by ~1e-3
(found tracing the round-1 2-rank CDP-v2 "deviation": one activation of the last
block at +1.07e-6 on the device and <= 0 here).  `Kinks` lets a caller supply the
device's own branch decisions (ReLU masks, max-pool argmaxes, read back from the
trainer after each step); they are used ONLY where this oracle's own value is
within `delta` of the switching point, everywhere else the float64 decision
stands.  `Kinks.used` counts the overridden elements.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F


class Kinks:
    """Device branch decisions for the ambiguous elements of one forward pass (see module doc).

    relu: list of bool arrays NCHW (device activation > 0) in forward ReLU order (stem, then per block
    the inner ReLUs and the output ReLU); pool: int array [B, C, Ho, Wo] of window indices r*3+s."""

    def __init__(self, relu=None, pool=None, delta=1e-5):
        self.relu, self.pool, self.delta = relu, pool, delta
        self.k = 0
        self.used = 0

    def relu_fn(self, v):
        if self.relu is None:
            return F.relu(v)
        dev = torch.from_numpy(np.asarray(self.relu[self.k]))
        self.k += 1
        m = v.detach() > 0
        amb = v.detach().abs() < self.delta
        self.used += int((amb & (m != dev)).sum())
        m = torch.where(amb, dev, m)
        return v * m.to(v.dtype)

    def pool_fn(self, y):
        if self.pool is None:
            return F.max_pool2d(y, 3, 2, 1)
        B, C, H, W = y.shape
        Ho, Wo = (H + 2 - 3) // 2 + 1, (W + 2 - 3) // 2 + 1
        yp = F.pad(y, (1, 1, 1, 1), value=float("-inf"))
        win = torch.stack([yp[:, :, r:r + 2 * Ho:2, s:s + 2 * Wo:2] for r in range(3) for s in range(3)], dim=2)
        best = win.detach().argmax(dim=2, keepdim=True)  # first maximum, as the device's strict '>' scan
        top = win.detach().gather(2, best)
        dev = torch.from_numpy(np.asarray(self.pool, dtype=np.int64)).unsqueeze(2)
        near = (top - win.detach().gather(2, dev)).abs() < self.delta
        self.used += int((near & (dev != best)).sum())
        idx = torch.where(near, dev, best)
        return win.gather(2, idx).squeeze(2)


def _relu(kinks, v):
    return F.relu(v) if kinks is None else kinks.relu_fn(v)


class Block(nn.Module):
    """BasicBlock (two 3x3) or Bottleneck (1x1, 3x3 with the stride, 1x1 x4; torchvision v1.5)."""

    def __init__(self, cin, width, stride, bottleneck=False):
        super().__init__()
        exp = 4 if bottleneck else 1
        cout = width * exp
        if bottleneck:
            shapes = [(cin, width, 1, 1), (width, width, 3, stride), (width, cout, 1, 1)]
        else:
            shapes = [(cin, width, 3, stride), (width, width, 3, 1)]
        self.convs = nn.ModuleList([nn.Conv2d(a, b, k, st, k // 2, bias=False) for a, b, k, st in shapes])
        self.bns = nn.ModuleList([nn.BatchNorm2d(b, eps=1e-5, track_running_stats=False) for _, b, _, _ in shapes])
        self.ds_conv = self.ds_bn = None
        if stride != 1 or cin != cout:
            self.ds_conv = nn.Conv2d(cin, cout, 1, stride, 0, bias=False)
            self.ds_bn = nn.BatchNorm2d(cout, eps=1e-5, track_running_stats=False)

    def forward(self, x, kinks=None):
        y = x
        n = len(self.convs)
        for i, (cv, bn) in enumerate(zip(self.convs, self.bns)):
            y = bn(cv(y))
            if i < n - 1:
                y = _relu(kinks, y)
        s = self.ds_bn(self.ds_conv(x)) if self.ds_conv is not None else x
        return _relu(kinks, y + s)


class TorchResNet(nn.Module):
    def __init__(self, widths=(64, 128, 256, 512), depths=(2, 2, 2, 2), classes=10, block="basic", stem="cifar"):
        super().__init__()
        self.imagenet = stem == "imagenet"
        if self.imagenet:
            self.stem_conv = nn.Conv2d(3, widths[0], 7, 2, 3, bias=False)
        else:
            self.stem_conv = nn.Conv2d(3, widths[0], 3, 1, 1, bias=False)
        self.stem_bn = nn.BatchNorm2d(widths[0], eps=1e-5, track_running_stats=False)
        bott = block == "bottleneck"
        exp = 4 if bott else 1
        blocks = []
        cin = widths[0]
        for l, (w, d) in enumerate(zip(widths, depths)):
            for k in range(d):
                blocks.append(Block(cin, w, 2 if (l > 0 and k == 0) else 1, bott))
                cin = w * exp
        self.blocks = nn.ModuleList(blocks)
        self.fc = nn.Linear(cin, classes)

    def forward(self, x, kinks=None):
        y = _relu(kinks, self.stem_bn(self.stem_conv(x)))
        if self.imagenet:
            y = F.max_pool2d(y, 3, 2, 1) if kinks is None else kinks.pool_fn(y)
        for b in self.blocks:
            y = b(y, kinks)
        return self.fc(y.mean(dim=(2, 3)))


CifarResNet = TorchResNet


def init_flat(widths, depths, seed=0, block="basic", stem="cifar", classes=10):
    """torch default initialisation under a fixed seed, exported to the trainer layout."""
    from paper_2403_08837_b200.resnet import torch_to_flat

    torch.manual_seed(seed)
    return torch_to_flat(TorchResNet(widths, depths, classes, block, stem))


def load_flat(model: TorchResNet, flat: np.ndarray, specs) -> None:
    from paper_2403_08837_b200.resnet import _ordered, flat_to_tensors

    parts = flat_to_tensors(flat, specs)
    with torch.no_grad():
        for (name, p), a, (kind, shape, _) in zip(_ordered(model), parts, specs):
            if kind == "conv":
                r, s, cin, cout = shape
                p.copy_(torch.from_numpy(np.ascontiguousarray(a.reshape(r, s, cin, cout).transpose(3, 2, 0, 1))))
            elif kind == "bn":
                c = shape[0] // 2
                p.pair[0].copy_(torch.from_numpy(a[:c]))
                p.pair[1].copy_(torch.from_numpy(a[c:]))
            else:
                rows, classes = shape
                m = a.reshape(rows, classes)
                p.pair[0].copy_(torch.from_numpy(np.ascontiguousarray(m[:-1].T)))
                p.pair[1].copy_(torch.from_numpy(m[-1]))


def grads_flat(model: TorchResNet, specs) -> list:
    """Gradients of the loaded parameters, per tensor, in the trainer layout."""
    from paper_2403_08837_b200.resnet import _ordered

    out = []
    for (name, p), (kind, shape, _) in zip(_ordered(model), specs):
        if kind == "conv":
            out.append(p.grad.detach().double().numpy().transpose(2, 3, 1, 0).ravel())
        elif kind == "bn":
            out.append(np.concatenate([p.pair[0].grad.double().numpy(), p.pair[1].grad.double().numpy()]))
        else:
            out.append(np.concatenate([p.pair[0].grad.double().numpy().T, p.pair[1].grad.double().numpy()[None, :]]).ravel())
    return out


class ResNetOracle:
    """value + per-tensor gradients of one micro-batch, float64 on the CPU."""

    def __init__(self, widths, depths, specs, block="basic", stem="cifar", classes=10, dtype=torch.float64):
        # dtype "bf16-autocast": float32 model under torch.autocast(bfloat16) (bf16 conv / linear
        # operands and outputs, float32 batch norm) — torch's own bf16 training step
        self.autocast = dtype == "bf16-autocast"
        if self.autocast:
            dtype = torch.float32
        self.model = TorchResNet(widths, depths, classes, block, stem).to(dtype)
        self.dtype = dtype
        self.specs = specs

    def loss_and_grads(self, params, x, y, kinks=None):
        load_flat(self.model, np.concatenate(params), self.specs)
        self.model.zero_grad(set_to_none=True)
        xt = torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float64).transpose(0, 3, 1, 2))).to(self.dtype)
        with torch.autocast("cpu", dtype=torch.bfloat16, enabled=self.autocast):
            z = self.model(xt, kinks)
        loss = F.cross_entropy(z.to(self.dtype), torch.from_numpy(np.asarray(y, np.int64)))
        loss.backward()
        return float(loss.item()), grads_flat(self.model, self.specs)


def run_cdp(widths, depths, init, inputs, labels, n_workers, micro_batch, perms, lr, momentum, fresh_tensor,
            block="basic", stem="cifar", classes=10, weight_decay=0.0, kinks=None, stats=None, dtype=None):
    """`steps = len(perms)` CDP steps from `init` (flat); fresh_tensor = N x n_tensors table (None = DP).

    dtype: the per-micro-batch forward / backward arithmetic (default float64; torch.float32 gives torch's
    own fp32 step, "bf16-autocast" its bf16 autocast step — the yardsticks for the device's fp32 / bf16
    tolerances at deep configurations); the accumulation and update stay float64 (oracle/engine.advance).

    kinks: optional kinks[t-1][i-1] -> Kinks (the device's branch decisions of worker i at step t);
    stats: optional dict, receives "kink_overrides" (elements where they were used)."""
    from oracle import engine as OE
    from paper_2403_08837_b200.resnet import flat_to_tensors, layer_specs

    hw = int(np.asarray(inputs).shape[1])
    specs = layer_specs(widths, depths, 3, hw, block, stem, classes)
    orc = ResNetOracle(widths, depths, specs, block, stem, classes, dtype or torch.float64)
    cur = [a.copy() for a in flat_to_tensors(np.asarray(init, np.float64), specs)]
    prev = [a.copy() for a in cur]
    vel = [np.zeros_like(a) for a in cur] if momentum else None
    losses = []
    used = 0
    for t, perm in enumerate(perms, start=1):
        batches = [(inputs[perm[i * micro_batch:(i + 1) * micro_batch]], labels[perm[i * micro_batch:(i + 1) * micro_batch]])
                   for i in range(n_workers)]
        grads_fn = orc.loss_and_grads
        if kinks is not None:
            worker = iter(range(n_workers))

            def grads_fn(params, x, y, _t=t, _w=worker):
                k = kinks[_t - 1][next(_w)]
                out = orc.loss_and_grads(params, x, y, k)
                nonlocal used
                used += k.used
                return out
        new, loss = OE.advance(None, cur, prev, t, batches, lr, fresh_tensor, momentum, vel,
                               weight_decay=weight_decay, grads_fn=grads_fn)
        prev, cur = cur, new
        losses.append(loss)
    if stats is not None:
        stats["kink_overrides"] = used
    return np.concatenate(cur), losses
