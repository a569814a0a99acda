"""Activation / state accounting for the hot-path schemes.

Only the rows of the reference cost model that the CDP step's memory claim
rests on (ref `pkg/src/cyclicdp/costs.py:111-119`, `:140-153`):

* single GPU: DP holds N*B*Psi_A of activations at peak, CDP (N+1)/2*B*Psi_A;
* multi GPU: B*Psi_A per device for both, but only CDP's *sum over devices*
  stays constant over the step;
* ZeRO state traffic per device per step: 2*Psi_P (DP broadcast) vs
  2(N-1)/N*Psi_P (CDP hops).

`activation_series` measures the same quantity from a plan (records live
from F.start through B.end, ref `costs.py:157-170`); the executor allocates
activation slots from exactly these intervals, so the planned peak is the
peak the device holds (checked against the device's own live-record
high-water counter in tests/test_gpu_vit_cyclic.py; the trainers allocate
with cudaMalloc, outside torch's caching allocator, so the bench reports the
trainer's allocated bytes beside it).  The analytic Table-1 reproduction and extrapolation
tooling (`costs.py:155-527`) are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .profiles import ModelProfile, ParallelismConfig, Scheme
from .schedule import TaskKind, Timeline


@dataclass(frozen=True)
class MemoryRow:
    activation_per_device: Fraction
    state_volume_per_device: Fraction


def closed_form_memory(cfg: ParallelismConfig, profile: ModelProfile) -> MemoryRow:
    if profile.n_stages != cfg.n:
        raise ValueError("profile stage count must equal n")
    n, b = cfg.n, cfg.micro_batch_size
    act = Fraction(b * profile.total_acts_per_sample)
    pp = profile.total_params
    s = cfg.scheme
    if s is Scheme.SINGLE_GPU_DP:
        return MemoryRow(n * act, Fraction(0))
    if s is Scheme.SINGLE_GPU_CDP:
        return MemoryRow(Fraction(n + 1, 2) * act, Fraction(0))
    if s in (Scheme.MULTI_GPU_DP, Scheme.MULTI_GPU_CDP):
        return MemoryRow(act, Fraction(0))
    if s is Scheme.ZERO_DP:
        return MemoryRow(act, Fraction(2 * pp))
    if s is Scheme.ZERO_CDP:
        return MemoryRow(act, Fraction(2 * (n - 1) * pp, n))
    raise NotImplementedError(f"scheme {s.value} is outside the hot path")


def activation_records(tl: Timeline) -> list:
    """(device, F.start, B.end, stage, micro_batch, step) per held record."""
    fwd: dict = {}
    out = []
    for t in tl.tasks:
        k = (t.micro_batch, t.stage, t.training_step)
        if t.kind is TaskKind.FORWARD:
            fwd[k] = t
            continue
        f = fwd.get(k)
        out.append((f.device if f else t.device, f.start if f else t.start, t.end, t.stage,
                    t.micro_batch, t.training_step))
    return out


def activation_series(tl: Timeline, profile: ModelProfile, per: str = "gpu") -> dict:
    """Live activation bytes per time step, keyed by gpu (or by device id)."""
    b = tl.cfg.micro_batch_size
    key_of = {d.id: (d.gpu if per == "gpu" else d.id) for d in tl.devices}
    delta: dict = {}
    for dev, lo, hi, stage, _i, _t in activation_records(tl):
        d = delta.setdefault(key_of[dev], [0] * (tl.horizon + 2))
        w = b * profile.stage_acts_per_sample[stage - 1]
        d[max(1, lo)] += w
        d[min(tl.horizon, hi) + 1] -= w
    out = {}
    for k, d in delta.items():
        acc, ser = 0, [0] * (tl.horizon + 1)
        for g in range(1, tl.horizon + 1):
            acc += d[g]
            ser[g] = acc
        out[k] = ser
    return out


def peak_activation(tl: Timeline, profile: ModelProfile) -> int:
    return max((max(s[1:], default=0) for s in activation_series(tl, profile).values()), default=0)
