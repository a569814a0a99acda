"""ORACLE — TEST INFRASTRUCTURE ONLY.  torch-CPU float64 restatement of the CDP step on Vision
Transformers (BASELINE configs[3]: ViT-B/16, 224x224).  The reference has no ViT, so
parity is "unpinned" by the reference: the reference's `_advance` semantics (oracle/engine.advance:
per-(micro-batch, stage) version choice, ascending accumulation, SGD-momentum update) applied to
per-micro-batch gradients computed here with torch autograd in float64.

Model (torchvision `vit_b_16` structure, written out so the device path can match it op for op):
patch embedding = conv(kernel = stride = patch), class token, learned position embedding, L pre-LN
encoder blocks (LN eps 1e-6; multi-head attention with a fused qkv projection in (q, k, v) order,
scores scaled by 1/sqrt(head_dim); MLP with exact-erf GELU), final LN, linear head on the class
token, softmax cross-entropy.  No dropout.

Flat parameter layout (paper_2403_08837_b200/vit.py, one hop unit per entry):
  patch [[W^T]; b] ([P*P*3 + 1][D], W row index (r*P + s)*3 + c), cls [D], pos [T][D],
  per block: ln1 [g | b], qkv [[W^T]; b] ([D+1][3D]), proj [[W^T]; b], ln2, fc1 [[W^T]; b] ([D+1][F]),
  fc2 [[W^T]; b] ([F+1][D]); final ln; head [[W^T]; b] ([D+1][classes]).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F


def vit_specs(image=224, patch=16, dim=768, depth=12, heads=12, mlp=3072, classes=1000):
    """[(name, shape)] of the flat parameter tensors, in order."""
    T = (image // patch) ** 2 + 1
    out = [("patch", (patch * patch * 3 + 1, dim)), ("cls", (dim,)), ("pos", (T, dim))]
    for i in range(depth):
        out += [(f"b{i}.ln1", (2 * dim,)), (f"b{i}.qkv", (dim + 1, 3 * dim)), (f"b{i}.proj", (dim + 1, dim)),
                (f"b{i}.ln2", (2 * dim,)), (f"b{i}.fc1", (dim + 1, mlp)), (f"b{i}.fc2", (mlp + 1, dim))]
    out += [("ln", (2 * dim,)), ("head", (dim + 1, classes))]
    return out


def init_flat(image=32, patch=8, dim=64, depth=2, heads=2, mlp=128, classes=10, seed=0):
    """Deterministic initialisation (numpy PCG64): linear weights N(0, 0.02), biases 0, LN (1, 0),
    cls / pos N(0, 0.02)."""
    rng = np.random.default_rng([seed, 0xF0])
    parts = []
    for name, shape in vit_specs(image, patch, dim, depth, heads, mlp, classes):
        n = int(np.prod(shape))
        if name.endswith(("ln1", "ln2")) or name == "ln":
            c = shape[0] // 2
            parts.append(np.concatenate([np.ones(c), np.zeros(c)]))
        elif name in ("cls", "pos"):
            parts.append(rng.normal(0.0, 0.02, size=n))
        else:
            rows, cols = shape
            w = rng.normal(0.0, 0.02, size=(rows - 1, cols))
            parts.append(np.concatenate([w, np.zeros((1, cols))]).ravel())
    return np.concatenate(parts)


def _split(flat, specs):
    out, pos = {}, 0
    for name, shape in specs:
        n = int(np.prod(shape))
        out[name] = flat[pos:pos + n].reshape(shape)
        pos += n
    return out


def vit_loss(flat: torch.Tensor, x: torch.Tensor, y: torch.Tensor, image, patch, dim, depth, heads, mlp, classes):
    """x: [B][H][W][3] (NHWC), y: [B] labels -> mean cross-entropy (float64 autograd graph)."""
    specs = vit_specs(image, patch, dim, depth, heads, mlp, classes)
    p = {}
    pos = 0
    for name, shape in specs:
        n = int(np.prod(shape))
        p[name] = flat[pos:pos + n].reshape(shape)
        pos += n
    B = x.shape[0]
    g = image // patch
    # patches [B*np][P*P*3], index (r*P + s)*3 + c
    xp = x.reshape(B, g, patch, g, patch, 3).permute(0, 1, 3, 2, 4, 5).reshape(B * g * g, patch * patch * 3)

    def lin(a, wb):
        return a @ wb[:-1] + wb[-1]

    def ln(a, gb):
        c = gb.shape[0] // 2
        return F.layer_norm(a, (c,), gb[:c], gb[c:], eps=1e-6)

    e = lin(xp, p["patch"]).reshape(B, g * g, dim)
    h = torch.cat([p["cls"].reshape(1, 1, dim).expand(B, 1, dim), e], dim=1) + p["pos"].unsqueeze(0)
    T = h.shape[1]
    hd = dim // heads
    for i in range(depth):
        u = ln(h, p[f"b{i}.ln1"])
        qkv = lin(u, p[f"b{i}.qkv"]).reshape(B, T, 3, heads, hd)
        q, k, v = qkv[:, :, 0].transpose(1, 2), qkv[:, :, 1].transpose(1, 2), qkv[:, :, 2].transpose(1, 2)
        s = (q @ k.transpose(-1, -2)) * (1.0 / math.sqrt(hd))
        a = torch.softmax(s, dim=-1) @ v
        h = h + lin(a.transpose(1, 2).reshape(B, T, dim), p[f"b{i}.proj"])
        u2 = ln(h, p[f"b{i}.ln2"])
        h = h + lin(F.gelu(lin(u2, p[f"b{i}.fc1"])), p[f"b{i}.fc2"])
    z = lin(ln(h[:, 0], p["ln"]), p["head"])
    return F.cross_entropy(z, y)


class VitOracle:
    def __init__(self, cfg):
        self.cfg = cfg
        self.specs = vit_specs(**cfg)
        self.sizes = [int(np.prod(s)) for _, s in self.specs]

    def loss_and_grads(self, params, x, y):
        flat = torch.tensor(np.concatenate(params), dtype=torch.float64, requires_grad=True)
        loss = vit_loss(flat, torch.from_numpy(np.asarray(x, np.float64)), torch.from_numpy(np.asarray(y, np.int64)),
                        **self.cfg)
        loss.backward()
        g = flat.grad.numpy()
        out, pos = [], 0
        for n in self.sizes:
            out.append(g[pos:pos + n].copy())
            pos += n
        return float(loss.item()), out


def run_cdp(cfg, init, inputs, labels, n_workers, micro_batch, perms, lr, momentum, fresh_tensor):
    """`len(perms)` CDP steps (fresh_tensor: N x n_tensors table, None = DP) -> (flat params, losses)."""
    from oracle import engine as OE

    orc = VitOracle(cfg)
    cur, pos = [], 0
    for n in orc.sizes:
        cur.append(np.asarray(init[pos:pos + n], np.float64).copy())
        pos += n
    prev = [a.copy() for a in cur]
    vel = [np.zeros_like(a) for a in cur] if momentum else None
    losses = []
    for t, perm in enumerate(perms, start=1):
        batches = [(inputs[perm[i * micro_batch:(i + 1) * micro_batch]], labels[perm[i * micro_batch:(i + 1) * micro_batch]])
                   for i in range(n_workers)]
        new, loss = OE.advance(None, cur, prev, t, batches, lr, fresh_tensor, momentum, vel,
                               grads_fn=orc.loss_and_grads)
        prev, cur = cur, new
        losses.append(loss)
    return np.concatenate(cur), losses
