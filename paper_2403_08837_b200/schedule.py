"""Task plans of one training step: DP lockstep, cyclic (CDP) and ZeRO placement.

Geometry (ref `pkg/src/cyclicdp/schedule.py:1-12`, `:148-151`, `:212-233`): a
step is a forward sweep over the N stages then the backward sweep, pass
length N*(fc+bc) time steps.  Under the cyclic schemes micro-batch i runs the
same pass shifted by 2*fc*(i-1).  Every task carries the parameter version it
reads, resolved through an `UpdateRule`.

This module is the *input* of the device executor: `cdp_b200` compiles a
Timeline into per-worker CUDA streams (one stream per `Device`), event edges
for the version / ring / activation-slot dependencies, and a CUDA graph per
training step (see `paper_2403_08837_b200/executor.py`).  Builders for the
model-partitioned schemes (MP, PP; ref `schedule.py:260-430`) are outside the
north-star path and raise.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from enum import Enum
from typing import Callable, Optional

from .events import CommEvent
from .profiles import ModelProfile, ParallelismConfig, Scheme
from .rules import UpdateRule, min_delay_rule, rule_by_name


class TaskKind(str, Enum):
    FORWARD = "F"
    BACKWARD = "B"


class ParamModel(str, Enum):
    REPLICA = "replica"
    RESIDENT = "resident"
    OWNED = "owned"


@dataclass(frozen=True)
class Device:
    id: str
    gpu: int
    capacity: Optional[int]
    param_model: ParamModel
    owned_stages: tuple = ()


@dataclass(frozen=True)
class Task:
    kind: TaskKind
    micro_batch: int
    stage: int
    training_step: int
    param_version: int
    device: str
    start: int
    duration: int = 1

    @property
    def end(self) -> int:
        return self.start + self.duration - 1

    def key(self) -> tuple:
        return (self.kind, self.micro_batch, self.stage, self.training_step)


def _task_order(t: Task):
    return (t.start, t.device)


def _event_order(e: CommEvent):
    return (e.boundary, e.src, e.stage)


@dataclass(frozen=True)
class Timeline:
    scheme: Scheme
    cfg: ParallelismConfig
    devices: tuple
    tasks: tuple
    comm_events: tuple
    horizon: int
    slots: dict = field(repr=False, hash=False, compare=False, default_factory=dict)

    @staticmethod
    def from_parts(scheme, cfg, devices, tasks, events=(), horizon=None) -> "Timeline":
        ordered = tuple(sorted(tasks, key=_task_order))
        if horizon is None:
            horizon = max((t.end for t in ordered), default=0)
        occupancy: dict = {}
        for t in ordered:
            for g in range(t.start, t.end + 1):
                occupancy.setdefault((t.device, g), t)
        return Timeline(
            scheme=scheme,
            cfg=cfg,
            devices=tuple(devices),
            tasks=ordered,
            comm_events=tuple(sorted(events, key=_event_order)),
            horizon=horizon,
            slots=occupancy,
        )

    def with_events(self, extra) -> "Timeline":
        return replace(self, comm_events=tuple(sorted(self.comm_events + tuple(extra), key=_event_order)))

    def device_by_id(self, device_id: str) -> Device:
        return next(d for d in self.devices if d.id == device_id)

    @property
    def n(self) -> int:
        return self.cfg.n

    @property
    def pass_length(self) -> int:
        w = self.cfg.cost_weights
        return self.n * (w.forward_cost + w.backward_cost)

    def steady_window(self) -> tuple:
        w = self.cfg.cost_weights
        lo = max(self.pass_length, 2 * w.forward_cost * (self.n - 1)) + 1
        return lo, self.pass_length * self.cfg.training_steps

    def task_index(self) -> dict:
        return {t.key(): t for t in self.tasks}

    def gpu_count(self) -> int:
        return len({d.gpu for d in self.devices})


def tree_depth(participants: int) -> int:
    """Dependent rounds of a tree collective (ref `schedule.py:138-140`)."""
    if participants <= 1:
        return 0
    return max(1, math.ceil(math.log2(participants)))


def stage_at_phase(phase: int, n: int) -> int:
    """Stage touched at local phase 1..2n of a unit-weight pass."""
    return phase if phase <= n else 2 * n + 1 - phase


def local_starts(n: int, fc: int, bc: int, j: int) -> tuple:
    """Offsets of F(j) and B(j) inside one pass (ref `schedule.py:148-151`)."""
    return (j - 1) * fc + 1, n * fc + (n - j) * bc + 1


def _need_scheme(cfg: ParallelismConfig, allowed) -> None:
    if cfg.scheme not in allowed:
        raise ValueError(f"scheme {cfg.scheme.value} not supported by this builder")


def resolve_rule(rule, n: int) -> UpdateRule:
    if isinstance(rule, str):
        rule = rule_by_name(rule, n)
    if rule.n != n:
        raise ValueError(f"rule is sized for n={rule.n}, config has n={n}")
    rule.check_feasible()
    return rule


def _workers(n: int, single: bool) -> list:
    return [
        Device(
            id=f"w{i}",
            gpu=0 if single else i - 1,
            capacity=None if single else n,
            param_model=ParamModel.RESIDENT if single else ParamModel.REPLICA,
        )
        for i in range(1, n + 1)
    ]


def _pass_tasks(cfg: ParallelismConfig, offset_of: Callable, version_of: Callable, device_of: Callable) -> list:
    """All F/B tasks of `cfg.training_steps` passes with per-(i,t) offsets."""
    n, w = cfg.n, cfg.cost_weights
    fc, bc = w.forward_cost, w.backward_cost
    plen = n * (fc + bc)
    out = []
    for t in range(1, cfg.training_steps + 1):
        for i in range(1, n + 1):
            base = (t - 1) * plen + offset_of(i)
            for j in range(1, n + 1):
                fs, bs = local_starts(n, fc, bc, j)
                v = version_of(i, j, t)
                d = device_of(i, j, t)
                out.append(Task(TaskKind.FORWARD, i, j, t, v, d, base + fs, fc))
                out.append(Task(TaskKind.BACKWARD, i, j, t, v, d, base + bs, bc))
    return out


def build_dp_timeline(cfg: ParallelismConfig) -> Timeline:
    """Lockstep baseline: every task of step t reads version t (ref `schedule.py:178-209`)."""
    _need_scheme(cfg, (Scheme.SINGLE_GPU_DP, Scheme.MULTI_GPU_DP))
    tasks = _pass_tasks(cfg, lambda i: 0, lambda i, j, t: t, lambda i, j, t: f"w{i}")
    w = cfg.cost_weights
    horizon = cfg.training_steps * cfg.n * (w.forward_cost + w.backward_cost)
    return Timeline.from_parts(cfg.scheme, cfg, _workers(cfg.n, cfg.scheme.is_single_gpu), tasks, horizon=horizon)


def cdp_tasks(cfg: ParallelismConfig, rule: UpdateRule, device_of: Callable) -> tuple:
    """Staggered tasks for every cyclic placement (ref `schedule.py:212-233`)."""
    stagger = 2 * cfg.cost_weights.forward_cost
    tasks = _pass_tasks(cfg, lambda i: stagger * (i - 1), rule.version_read, device_of)
    w = cfg.cost_weights
    horizon = cfg.training_steps * cfg.n * (w.forward_cost + w.backward_cost) + stagger * (cfg.n - 1)
    return tasks, horizon


def build_cdp_timeline(cfg: ParallelismConfig, rule="cdp-v2") -> Timeline:
    """Cyclic plan, micro-batch i on worker i (ref `schedule.py:236-257`)."""
    _need_scheme(cfg, (Scheme.SINGLE_GPU_CDP, Scheme.MULTI_GPU_CDP))
    rule = resolve_rule(rule, cfg.n)
    tasks, horizon = cdp_tasks(cfg, rule, lambda i, j, t: f"w{i}")
    return Timeline.from_parts(cfg.scheme, cfg, _workers(cfg.n, cfg.scheme.is_single_gpu), tasks, horizon=horizon)


def build_zero_timeline(cfg: ParallelismConfig, profile: ModelProfile, cyclic: bool) -> Timeline:
    """State-sharded placement: w_i owns stage i's states (ref `schedule.py:433-472`)."""
    _need_scheme(cfg, (Scheme.ZERO_DP, Scheme.ZERO_CDP))
    if cyclic != (cfg.scheme is Scheme.ZERO_CDP):
        raise ValueError("cyclic flag does not match the configured scheme")
    if not cfg.cost_weights.is_unit:
        raise ValueError("state-sharded builders require unit cost weights")
    if profile.n_stages != cfg.n:
        raise ValueError("profile stage count must equal n")
    n = cfg.n
    devices = [
        Device(id=f"w{i}", gpu=i - 1, capacity=n, param_model=ParamModel.OWNED, owned_stages=(i,))
        for i in range(1, n + 1)
    ]
    if cyclic:
        tasks, horizon = cdp_tasks(cfg, min_delay_rule(n), lambda i, j, t: f"w{i}")
        return Timeline.from_parts(cfg.scheme, cfg, devices, tasks, horizon=horizon)
    tasks = _pass_tasks(cfg, lambda i: 0, lambda i, j, t: t, lambda i, j, t: f"w{i}")
    return Timeline.from_parts(cfg.scheme, cfg, devices, tasks, horizon=cfg.training_steps * 2 * n)


def build_pp_timeline(*_a, **_k):
    raise NotImplementedError("pipeline placement is outside the CDP data-parallel hot path (DESIGN.md §Scope)")


def build_mp_timeline(*_a, **_k):
    raise NotImplementedError("model-partitioned placement is outside the CDP data-parallel hot path (DESIGN.md §Scope)")


@dataclass(frozen=True)
class Violation:
    kind: str
    message: str


@dataclass(frozen=True)
class ValidationReport:
    violations: tuple

    @property
    def ok(self) -> bool:
        return not self.violations

    def by_kind(self, kind: str) -> list:
        return [v for v in self.violations if v.kind == kind]


def version_ready_times(tl: Timeline) -> dict:
    """(stage, version) -> last time step of the backward contributions that produce it."""
    ready: dict = {}
    for t in tl.tasks:
        if t.kind is TaskKind.BACKWARD:
            key = (t.stage, t.training_step + 1)
            if t.end > ready.get(key, 0):
                ready[key] = t.end
    return ready


def activation_intervals(tl: Timeline) -> dict:
    """(i, j, t) -> [device, F.start, B.end or None]; the record lives F.start..B.end."""
    rec: dict = {}
    for t in tl.tasks:
        key = (t.micro_batch, t.stage, t.training_step)
        if t.kind is TaskKind.FORWARD:
            rec.setdefault(key, [t.device, t.start, None])
        elif key in rec:
            rec[key][2] = t.end
    return rec


def validate_timeline(tl: Timeline) -> ValidationReport:
    """Dependency legality, reported as data (ref `schedule.py:493-600`).

    Kinds: device-conflict, forward-order, forward-before-backward,
    activation-locality, backward-order, stale-read, capacity.
    """
    out: list = []
    idx = tl.task_index()

    held: dict = {}
    for t in tl.tasks:
        for g in range(t.start, t.end + 1):
            prior = held.get((t.device, g))
            if prior is not None and prior is not t:
                out.append(Violation("device-conflict", f"device {t.device} runs two tasks at step {g}"))
            else:
                held[(t.device, g)] = t

    for t in tl.tasks:
        i, j, s = t.micro_batch, t.stage, t.training_step
        if t.kind is TaskKind.FORWARD:
            if j > 1:
                p = idx.get((TaskKind.FORWARD, i, j - 1, s))
                if p is None or p.end >= t.start:
                    out.append(Violation("forward-order", f"forward ({i},{j},{s}) not preceded by stage {j - 1}"))
            continue
        f = idx.get((TaskKind.FORWARD, i, j, s))
        if f is None or f.end >= t.start:
            out.append(Violation("forward-before-backward", f"backward ({i},{j},{s}) precedes its forward"))
        elif f.device != t.device:
            out.append(
                Violation(
                    "activation-locality",
                    f"backward ({i},{j},{s}) runs on {t.device} but its forward ran on {f.device}",
                )
            )
        if j < tl.n:
            nx = idx.get((TaskKind.BACKWARD, i, j + 1, s))
            if nx is None or nx.end >= t.start:
                out.append(Violation("backward-order", f"backward ({i},{j},{s}) not preceded by stage {j + 1}"))

    ready = version_ready_times(tl)
    for t in tl.tasks:
        v = t.param_version
        if v <= 1:
            continue
        r = ready.get((t.stage, v))
        who = f"task ({t.micro_batch},{t.stage},{t.training_step}) reads version {v}"
        if r is None:
            out.append(Violation("stale-read", f"{who} that is never produced"))
        elif t.start <= r:
            out.append(Violation("stale-read", f"{who} at step {t.start}, available only after step {r}"))

    per_dev: dict = {}
    for dev, lo, hi in activation_intervals(tl).values():
        per_dev.setdefault(dev, []).append((lo, tl.horizon if hi is None else hi))
    for d in tl.devices:
        if d.capacity is None:
            continue
        delta: dict = {}
        for lo, hi in per_dev.get(d.id, ()):
            delta[lo] = delta.get(lo, 0) + 1
            delta[hi + 1] = delta.get(hi + 1, 0) - 1
        live = 0
        for g in sorted(delta):
            live += delta[g]
            if live > d.capacity:
                out.append(
                    Violation(
                        "capacity",
                        f"device {d.id} holds {live} activation records at step {g}, capacity {d.capacity}",
                    )
                )
                break
    return ValidationReport(tuple(out))
