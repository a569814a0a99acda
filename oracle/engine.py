"""ORACLE — TEST INFRASTRUCTURE ONLY.  fp64 restatement of the CDP step.

* `advance`         ref `pkg/src/cyclicdp/training/engine.py:66-116`
                    (per-micro-batch version choice by rule, ascending-i
                    accumulation, SGD / SGD+momentum update)
* `run_experiment`  ref `engine.py:168-215` (same init + data order per rule,
                    divergence detection)
* `make_mlp_task`, `make_quadratic_task`, `micro_batches`, `init_params`
                    ref `training/models.py:70-77`, `:136-140`, `:173-225`
                    (numpy PCG64 streams keyed exactly like the reference)

`weight_decay` is an extension the reference lacks (SURVEY §7 hard part 5):
g = acc/n + wd*theta_t; with momentum v = m*v + g, theta' = theta_t - lr*v;
without, theta' = theta_t - lr*g.  wd = 0 reproduces the reference formulas
exactly, so parity against the reference is pinned at wd = 0 only.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import kernels as K


# ----------------------------------------------------------------- rules
def fresh_table(rule: str, n: int):
    if rule == "dp":
        return None
    if rule in ("cdp-v1", "v1"):
        return [[False] * n for _ in range(n)]
    if rule in ("cdp-v2", "v2"):
        return [[i + j >= n + 1 for j in range(1, n + 1)] for i in range(1, n + 1)]
    raise ValueError(rule)


# ----------------------------------------------------------------- tasks
@dataclass
class MlpTask:
    dims: tuple
    loss_kind: str
    inputs: np.ndarray
    targets: np.ndarray
    n: int
    micro_batch_size: int
    seed: int

    @property
    def stage_sizes(self):
        return tuple(self.dims[j] * self.dims[j + 1] + self.dims[j + 1] for j in range(len(self.dims) - 1))

    def init_params(self):
        return mlp_init(self.dims, np.random.default_rng([self.seed, 0xC0]))

    def micro_batches(self, step: int):
        perm = np.random.default_rng([self.seed, step]).permutation(len(self.inputs))
        b = self.micro_batch_size
        return [(self.inputs[perm[i * b:(i + 1) * b]], self.targets[perm[i * b:(i + 1) * b]]) for i in range(self.n)]

    def loss_and_grads(self, stage_params, x, y):
        theta = np.concatenate(stage_params)
        if self.loss_kind == "mse":
            loss, g = K.mlp_value_grad(self.dims, theta, x, y, None, 0)
        else:
            loss, g = K.mlp_value_grad(self.dims, theta, x, None, y.astype(np.int64), 1)
        return loss, split(g, self.stage_sizes)


def split(flat, sizes):
    out, pos = [], 0
    for s in sizes:
        out.append(flat[pos:pos + s])
        pos += s
    return out


def mlp_init(dims, rng):
    out = []
    for j in range(len(dims) - 1):
        din, dout = dims[j], dims[j + 1]
        w = rng.normal(0.0, 1.0 / np.sqrt(din), size=din * dout)
        out.append(np.concatenate([w, np.zeros(dout)]))
    return out


def mlp_forward(dims, params, x):
    h = x
    for j in range(len(dims) - 1):
        din, dout = dims[j], dims[j + 1]
        w = params[j][: din * dout].reshape(din, dout)
        h = h @ w + params[j][din * dout:]
        if j < len(dims) - 2:
            h = np.tanh(h)
    return h


def make_mlp_task(n, micro_batch_size=2, seed=0, width=6, in_dim=4, out_dim=2, loss_kind="mse", noise=0.05):
    dims = (in_dim,) + (width,) * (n - 1) + (out_dim,)
    rng = np.random.default_rng([seed, 0xB0])
    size = n * micro_batch_size
    x = rng.normal(0.0, 1.0, size=(size, in_dim))
    teacher = mlp_init(dims, np.random.default_rng([seed, 0xB1]))
    clean = mlp_forward(dims, teacher, x)
    if loss_kind == "mse":
        tgt = clean + noise * rng.normal(size=clean.shape)
    else:
        tgt = np.argmax(clean, axis=1).astype(np.int64)
    return MlpTask(dims, loss_kind, x, tgt, n, micro_batch_size, seed)


@dataclass
class QuadTask:
    a: np.ndarray
    stage_sizes: tuple
    inputs: np.ndarray
    targets: np.ndarray
    n: int
    micro_batch_size: int
    seed: int

    def init_params(self):
        rng = np.random.default_rng([self.seed, 0xC0])
        return [rng.normal(0.0, 1.0, size=s) for s in self.stage_sizes]

    micro_batches = MlpTask.micro_batches

    def loss_and_grads(self, stage_params, x, y):
        loss, g = K.quad_value_grad(self.a, np.concatenate(stage_params), y)
        return loss, split(g, self.stage_sizes)


def make_quadratic_task(n, micro_batch_size=2, seed=0, dim_per_stage=3, eig_low=0.5, eig_high=1.5):
    rng = np.random.default_rng([seed, 0xA0])
    dim = n * dim_per_stage
    q, _ = np.linalg.qr(rng.normal(size=(dim, dim)))
    a = np.diag(np.sqrt(np.linspace(eig_low, eig_high, dim) * dim)) @ q
    size = n * micro_batch_size
    targets = rng.normal(0.0, 1.0, size=(size, a.shape[0]))
    return QuadTask(a, (dim_per_stage,) * n, np.zeros((size, 1)), targets, n, micro_batch_size, seed)


# ----------------------------------------------------------------- engine
class OracleDiverged(RuntimeError):
    def __init__(self, stage):
        self.stage = stage
        super().__init__(f"non-finite at stage {stage}")


def advance(task, current, previous, step, batches, lr, fresh, momentum=0.0, velocity=None,
            weight_decay=0.0, trace=None, grads_fn=None):
    """One training step; returns (new_current, mean_loss).  `fresh` None = DP."""
    n = len(batches)
    acc = None
    loss_sum = 0.0
    for i in range(1, n + 1):
        if fresh is None:
            params = current
            versions = [step] * len(current)
        else:
            params = [current[j] if fresh[i - 1][j] else previous[j] for j in range(len(current))]
            versions = [step if fresh[i - 1][j] else step - 1 for j in range(len(current))]
        if trace is not None:
            trace.extend((step, i, j + 1, v) for j, v in enumerate(versions))
        x, y = batches[i - 1]
        loss, g = (grads_fn or task.loss_and_grads)(params, x, y)
        for jj, gg in enumerate(g, start=1):
            if not np.all(np.isfinite(gg)):
                raise OracleDiverged(jj)
        if not np.isfinite(loss):
            raise OracleDiverged(0)
        loss_sum += loss
        if acc is None:
            acc = [gg.copy() for gg in g]
        else:
            for a, gg in zip(acc, g):
                a += gg
    if weight_decay:
        acc = [a / n + weight_decay * c for a, c in zip(acc, current)]
        scale_done = True
    else:
        scale_done = False
    if momentum and velocity is not None:
        for v, a in zip(velocity, acc):
            v *= momentum
            v += a if scale_done else a / n
        new = [c - lr * v for c, v in zip(current, velocity)]
    elif scale_done:
        new = [c - lr * a for c, a in zip(current, acc)]
    else:
        new = [c - (lr / n) * a for c, a in zip(current, acc)]
    for j, p in enumerate(new, start=1):
        if not np.all(np.isfinite(p)):
            raise OracleDiverged(j)
    return new, loss_sum / n


@dataclass
class OracleRun:
    rule: str
    losses: list = field(default_factory=list)
    final_params: Optional[list] = None
    diverged_at: Optional[int] = None
    trace: Optional[list] = None


def run_experiment(task, rules=("dp", "cdp-v1", "cdp-v2"), steps=100, lr=0.1, momentum=0.0,
                   record_trace=False, divergence_limit=1e12, weight_decay=0.0):
    lr_of: Callable = lr if callable(lr) else (lambda t: lr)
    out = {}
    for rule in rules:
        fresh = fresh_table(rule, task.n)
        init = task.init_params()
        cur = [p.copy() for p in init]
        prev = [p.copy() for p in init]
        vel = [np.zeros_like(p) for p in cur] if momentum else None
        run = OracleRun(rule, trace=[] if record_trace else None)
        for t in range(1, steps + 1):
            try:
                new, loss = advance(task, cur, prev, t, task.micro_batches(t), lr_of(t), fresh,
                                    momentum, vel, weight_decay, run.trace)
            except OracleDiverged:
                run.diverged_at = t
                break
            prev, cur = cur, new
            run.losses.append(loss)
            if not np.isfinite(loss) or abs(loss) > divergence_limit:
                run.diverged_at = t
                break
        run.final_params = cur
        out[rule] = run
    return out
