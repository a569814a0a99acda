"""Training step API (drop-in for ref `training/engine.py:1-238`).

Same names, signatures and version convention as the reference: theta_1 is
the initialisation, step t produces version t+1, stale reads at t = 1 see
version 0, an alias of the initialisation (ref `engine.py:8-10`).

For `StageMlp` models every step runs on the device: `run_experiment`
keeps one `DeviceMlpTrainer` per rule resident across steps (parameters,
momentum, data and both step graphs stay in HBM; only the step's
permutation and learning rate travel), and `step_dp` / `step_cdp` /
`_advance` run one device step from the given host state.  Other models
(the coupled-quadratic fixture) evaluate their per-micro-batch gradients
through the backend operator and accumulate in the reference order.

Extensions over the reference, all defaulting to its behaviour:
`dtype` ("fp32" = 3xTF32 tensor-core products, fp32 master state; "bf16" =
bf16 operands, fp32 accumulate and master state) and `weight_decay`
(g = acc/n + wd*theta_t; 0 reproduces the reference formulas).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence, Union

import numpy as np

from ..rules import UpdateRule, max_delay_rule, min_delay_rule
from ..schedule import TaskKind, Timeline
from .models import NonFiniteGradientError, StageMlp, ToyTask, split_stages

RULE_DP = "dp"


@dataclass
class VersionedParams:
    """theta_t (`current`), theta_{t-1} (`previous`), `step` = t."""

    current: list
    previous: list
    step: int

    @staticmethod
    def initial(params: Sequence[np.ndarray]) -> "VersionedParams":
        return VersionedParams([p.copy() for p in params], [p.copy() for p in params], 1)


def grad_stagewise(model, stage_params, batch):
    x, y = batch
    return model.loss_and_grads(stage_params, x, y)


def _resolve_rule(rule: Union[str, UpdateRule], n: int) -> Optional[UpdateRule]:
    """ref `engine.py:51-63`."""
    if isinstance(rule, UpdateRule):
        if rule.n != n:
            raise ValueError("rule size does not match task")
        rule.check_feasible()
        return rule
    if rule == RULE_DP:
        return None
    if rule in ("cdp-v1", "v1"):
        return max_delay_rule(n)
    if rule in ("cdp-v2", "v2"):
        return min_delay_rule(n)
    raise ValueError(f"unknown rule {rule!r}")


def _versions(rule: Optional[UpdateRule], i: int, n_stages: int, t: int) -> list:
    if rule is None:
        return [t] * n_stages
    return [rule.version_read(i, j, t) for j in range(1, n_stages + 1)]


def raise_for_flags(flags) -> None:
    """Map device non-finite flags to the reference exception (ref models.py:29-34, engine.py:110-112)."""
    grad, loss, upd = (int(f) for f in flags)
    if grad:
        raise NonFiniteGradientError((grad & -grad).bit_length())
    if loss:
        raise NonFiniteGradientError(0, "loss")
    if upd:
        raise NonFiniteGradientError((upd & -upd).bit_length(), "update")


# ----------------------------------------------------------------------------- device path
_TRAINERS: dict = {}


def _device_trainer(model: StageMlp, n: int, b: int, rule, dtype: str, momentum: float, wd: float):
    from ..device import DeviceMlpTrainer

    key = (model.dims, model.loss_kind, n, b, None if rule is None else rule.fresh, dtype, float(momentum), float(wd))
    tr = _TRAINERS.get(key)
    if tr is None:
        tr = DeviceMlpTrainer(model.dims, b, n, model.loss_code, rule, dtype=dtype, momentum=momentum,
                              weight_decay=wd)
        _TRAINERS[key] = tr
    return tr


def _advance_device(model: StageMlp, state: VersionedParams, batches, lr, rule, trace, momentum, velocity, wd, dtype):
    n = len(batches)
    b = len(batches[0][0])
    use_mom = bool(momentum) and velocity is not None
    tr = _device_trainer(model, n, b, rule, dtype, momentum if use_mom else 0.0, wd)
    t = state.step
    if trace is not None:
        for i in range(1, n + 1):
            trace.extend((t, i, j, v) for j, v in enumerate(_versions(rule, i, len(state.current), t), start=1))
    tr.set_params(np.concatenate(state.current), which=0)
    tr.set_params(np.concatenate(state.previous), which=1)
    if use_mom:
        tr.set_velocity(np.concatenate(velocity))
    x = np.concatenate([bt[0] for bt in batches])
    y = np.concatenate([bt[1] for bt in batches])
    tr.step_host_batch(x, y, lr)
    losses, flags = tr.history(1)
    raise_for_flags(flags[-1])
    new = split_stages(tr.get_params(0).astype(np.float64), model.stage_sizes)
    if use_mom:
        for v, nv in zip(velocity, split_stages(tr.get_velocity().astype(np.float64), model.stage_sizes)):
            v[...] = nv
    return VersionedParams(current=new, previous=state.current, step=t + 1), float(losses[-1])


def _advance_host(model, state, batches, lr, rule, trace, momentum, velocity, wd):
    """Per-micro-batch gradients from the GPU operator, reference accumulation order."""
    n = len(batches)
    t = state.step
    acc = None
    loss_sum = 0.0
    for i in range(1, n + 1):
        if rule is None:
            params = state.current
        else:
            params = [state.current[j - 1] if rule.reads_fresh(i, j) else state.previous[j - 1]
                      for j in range(1, len(state.current) + 1)]
        if trace is not None:
            trace.extend((t, i, j, v) for j, v in enumerate(_versions(rule, i, len(state.current), t), start=1))
        loss, grads = grad_stagewise(model, params, batches[i - 1])
        loss_sum += loss
        if acc is None:
            acc = [g.copy() for g in grads]
        else:
            for a, g in zip(acc, grads):
                a += g
    if wd:
        acc = [a / n + wd * c for a, c in zip(acc, state.current)]
    if momentum and velocity is not None:
        for v, a in zip(velocity, acc):
            v *= momentum
            v += a if wd else a / n
        new = [c - lr * v for c, v in zip(state.current, velocity)]
    elif wd:
        new = [c - lr * a for c, a in zip(state.current, acc)]
    else:
        new = [c - (lr / n) * a for c, a in zip(state.current, acc)]
    for j, p in enumerate(new, start=1):
        if not np.all(np.isfinite(p)):
            raise NonFiniteGradientError(j, "update")
    return VersionedParams(current=new, previous=state.current, step=t + 1), loss_sum / n


def _advance(model, state: VersionedParams, batches, lr: float, rule: Optional[UpdateRule], trace: Optional[list],
             momentum: float = 0.0, velocity: Optional[list] = None, weight_decay: float = 0.0,
             dtype: str = "fp32"):
    """One training step (ref `engine.py:66-116`)."""
    if isinstance(model, StageMlp):
        return _advance_device(model, state, batches, lr, rule, trace, momentum, velocity, weight_decay, dtype)
    return _advance_host(model, state, batches, lr, rule, trace, momentum, velocity, weight_decay)


def step_dp(model, state: VersionedParams, batches, lr: float, dtype: str = "fp32"):
    """Synchronous step: every micro-batch at the current version (ref `engine.py:119-122`)."""
    return _advance(model, state, batches, lr, rule=None, trace=None, dtype=dtype)


def step_cdp(model, state: VersionedParams, batches, lr: float, rule: Union[str, UpdateRule], dtype: str = "fp32"):
    """Cyclic step under `rule` (ref `engine.py:125-134`)."""
    resolved = _resolve_rule(rule, len(batches))
    if resolved is None:
        raise ValueError("use step_dp for the synchronous rule")
    return _advance(model, state, batches, lr, rule=resolved, trace=None, dtype=dtype)


@dataclass
class RuleRun:
    rule: str
    losses: list = field(default_factory=list)
    final_params: Optional[list] = None
    diverged_at: Optional[int] = None
    trace: Optional[list] = None


@dataclass
class ExperimentResult:
    runs: dict
    steps: int
    seed: int

    def final_losses(self) -> dict:
        return {name: run.losses[-1] for name, run in self.runs.items() if run.losses}

    def max_pairwise_divergence(self) -> float:
        names = list(self.runs)
        worst = 0.0
        for a in range(len(names)):
            for b in range(a + 1, len(names)):
                for va, vb in zip(self.runs[names[a]].losses, self.runs[names[b]].losses):
                    worst = max(worst, abs(va - vb))
        return worst


def _first_divergence(losses, flags, limit):
    """(step, kind): kind 'flag' (exception in the reference) or 'loss'."""
    for k in range(len(losses)):
        if flags[k].any():
            return k + 1, "flag"
        if not np.isfinite(losses[k]) or abs(losses[k]) > limit:
            return k + 1, "loss"
    return None, None


def _run_device(task: ToyTask, rule, steps, lr_of, momentum, wd, dtype, limit):
    from ..device import DeviceMlpTrainer

    model: StageMlp = task.model

    def fresh_trainer():
        tr = DeviceMlpTrainer(model.dims, task.micro_batch_size, task.n, model.loss_code, rule, dtype=dtype,
                              momentum=momentum, weight_decay=wd, inputs=task.inputs, targets=task.targets)
        tr.set_params(np.concatenate(task.init_params()), which=-1)
        return tr

    def run(tr, k):
        for t in range(1, k + 1):
            tr.step(task.permutation(t), lr_of(t))
        return tr.history(k)

    tr = fresh_trainer()
    losses, flags = run(tr, steps)
    d, kind = _first_divergence(losses, flags, limit)
    if d is None:
        final = tr.get_params(0)
        kept = list(losses)
        last = steps
    else:
        kept = list(losses[: d - 1] if kind == "flag" else losses[:d])
        last = d
        tr.close()
        tr = fresh_trainer()  # deterministic replay up to the state the reference returns
        run(tr, d - 1 if kind == "flag" else d)
        final = tr.get_params(0)
    tr.close()
    return kept, split_stages(final.astype(np.float64), model.stage_sizes), d, last


def run_experiment(task: ToyTask, rules=(RULE_DP, "cdp-v1", "cdp-v2"), steps: int = 100,
                   lr: Union[float, Callable[[int], float]] = 0.1, momentum: float = 0.0,
                   record_trace: bool = False, divergence_limit: float = 1e12, dtype: str = "fp32",
                   weight_decay: float = 0.0) -> ExperimentResult:
    """Every rule from the same initialisation and data order (ref `engine.py:168-215`)."""
    lr_of = lr if callable(lr) else (lambda t: lr)
    runs = {}
    for rule in rules:
        name = rule if isinstance(rule, str) else rule.name
        resolved = _resolve_rule(rule, task.n) if name != RULE_DP else None
        run = RuleRun(rule=name, trace=[] if record_trace else None)
        if isinstance(task.model, StageMlp):
            run.losses, run.final_params, run.diverged_at, last = _run_device(
                task, resolved, steps, lr_of, momentum, weight_decay, dtype, divergence_limit)
            if record_trace:
                for t in range(1, last + 1):
                    for i in range(1, task.n + 1):
                        run.trace.extend((t, i, j, v) for j, v in
                                         enumerate(_versions(resolved, i, task.model.n_stages, t), start=1))
        else:
            state = VersionedParams.initial(task.init_params())
            velocity = [np.zeros_like(p) for p in state.current] if momentum else None
            for t in range(1, steps + 1):
                try:
                    state, loss = _advance(task.model, state, task.micro_batches(t), lr_of(t), resolved, run.trace,
                                           momentum, velocity, weight_decay, dtype)
                except NonFiniteGradientError:
                    run.diverged_at = t
                    break
                run.losses.append(loss)
                if not np.isfinite(loss) or abs(loss) > divergence_limit:
                    run.diverged_at = t
                    break
            run.final_params = state.current
        runs[name] = run
    return ExperimentResult(runs=runs, steps=steps, seed=task.seed)


def schedule_consistency_check(tl: Timeline, trace: Sequence[tuple]):
    """Engine trace vs FORWARD tasks' param_version (ref `engine.py:218-238`)."""
    expected = {(t.training_step, t.micro_batch, t.stage): t.param_version
                for t in tl.tasks if t.kind is TaskKind.FORWARD}
    for t, i, j, version in trace:
        want = expected.get((t, i, j))
        if want is not None and want != version:
            return False, (t, i, j, version, want)
    return True, None
