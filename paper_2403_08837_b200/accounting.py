"""Activation and communication accounting on EXECUTED schedules.

The reference tallies memory and communication from a planned timeline
(`measure_costs`, ref `costs.py:191-329`; `balance_report`, ref
`comm.py:196-221`).  This module computes the same fields from the schedule
the GPU actually ran: per-task %globaltimer stamps taken by the device around
every forward / backward (`DeviceMlpTrainer.trace_step`, `cli trace`), keyed
`(TaskKind, micro_batch, stage, step) -> (start_ns, end_ns)`.

* Activation records (ref `costs.py:157-170`): the record of (i, j, t) is
  live from the start of F(i, j, t) to the end of B(i, j, t); its size is the
  device's own record bytes for stage j.  The executed live-bytes series is a
  step function over device time; its peak, its range over the steady window
  and its time average are the measured counterparts of
  `peak_activation_memory_per_device`, `steady_activation_*`.
* Gradient hops (ref `comm.py:37-67`): B(i, j, t) sends stage j's partial sum
  w_i -> w_{i+1} when it ends.  Each executed hop is attributed to the plan
  boundary of its task; per boundary the sends / receives histogram of
  `balance_report` is rebuilt from the executed hops, and the chain order
  (hop i after hop i-1 of the same (j, t)) is checked on device time.
"""

from __future__ import annotations

from dataclasses import dataclass

from .schedule import TaskKind, Timeline


@dataclass(frozen=True)
class ExecutedActivation:
    peak_bytes: int          # max live bytes over device time
    steady_max_bytes: int    # max over the steady window (steps 2 .. T-1 of the run)
    steady_min_bytes: int    # min over the steady window
    mean_bytes: float        # time-weighted mean over the steady window
    window_ns: int           # length of the steady window


def executed_records(executed: dict) -> list:
    """(micro_batch, stage, step, F.start_ns, B.end_ns) per activation record."""
    out = []
    for (kind, i, j, t), (s, e) in executed.items():
        if kind is not TaskKind.BACKWARD:
            continue
        f = executed.get((TaskKind.FORWARD, i, j, t))
        if f is None:
            raise ValueError(f"backward ({i},{j},{t}) has no executed forward")
        out.append((i, j, t, f[0], e))
    return out


def activation_series_ns(executed: dict, record_bytes) -> list:
    """[(time_ns, live_bytes)] change points of the executed live-activation series; record_bytes[j-1] is
    the device's record size for stage j.  A record is released before one acquired at the same instant."""
    ev = []
    for i, j, t, lo, hi in executed_records(executed):
        w = int(record_bytes[j - 1])
        ev.append((lo, 1, w))
        ev.append((hi, 0, -w))
    ev.sort()
    out, live = [], 0
    for tns, _order, d in ev:
        live += d
        if out and out[-1][0] == tns:
            out[-1] = (tns, live)
        else:
            out.append((tns, live))
    return out


def executed_activation(executed: dict, record_bytes, steps: int) -> ExecutedActivation:
    """Measured activation fields of a run of `steps` training steps (steady window: from the first task of
    step 2 to the last task of step steps - 1; needs steps >= 3, as ref measure_costs)."""
    if steps < 3:
        raise ValueError("measurement needs >= 3 executed training steps")
    ser = activation_series_ns(executed, record_bytes)
    lo = min(s for (k, i, j, t), (s, e) in executed.items() if t == 2)
    hi = max(e for (k, i, j, t), (s, e) in executed.items() if t == steps - 1)
    peak = max(v for _, v in ser)
    inside, area = [], 0.0
    live = 0
    prev_t = lo
    for tns, v in ser:
        if tns <= lo:
            live = v
            continue
        if tns > hi:
            break
        inside.append(live)
        area += live * (tns - prev_t)
        prev_t, live = tns, v
    inside.append(live)
    area += live * (hi - prev_t)
    return ExecutedActivation(peak, max(inside), min(inside), area / max(hi - lo, 1), hi - lo)


def executed_hops(executed: dict, n: int) -> list:
    """(stage, step, src worker, dst worker, t_ns) of every gradient hop (B(i, j, t) end, i < ... ring:
    w_i -> w_{i mod n + 1}, ref comm.py:52-66)."""
    out = []
    for (kind, i, j, t), (s, e) in executed.items():
        if kind is TaskKind.BACKWARD:
            out.append((j, t, i, i % n + 1, e))
    return sorted(out, key=lambda h: h[4])


def executed_balance(tl: Timeline, executed: dict) -> dict:
    """balance_report over the executed hops: each hop is attributed to its plan task's boundary (B.end);
    returns the per-boundary sends / receives histogram (max, min, mean sends; every worker sends and
    receives at most one hop per boundary, ref comm.py:37-67) and the chain-order violations measured on
    device time (a hop of w_i completing before the hop of w_{i-1} for the same stage and step)."""
    n = tl.n
    plan_end = {(t.kind, t.micro_batch, t.stage, t.training_step): t.end for t in tl.tasks}
    per = {}
    for j, t, src, dst, _tns in executed_hops(executed, n):
        b = plan_end[(TaskKind.BACKWARD, src, j, t)]
        d = per.setdefault(b, {"sends": {}, "recvs": {}})
        d["sends"][src] = d["sends"].get(src, 0) + 1
        d["recvs"][dst] = d["recvs"].get(dst, 0) + 1
    counts = [sum(d["sends"].values()) for d in per.values()] or [0]
    max_per_worker = max((max(max(d["sends"].values()), max(d["recvs"].values())) for d in per.values()),
                         default=0)
    order = []
    hop_t = {(j, t, src): tns for j, t, src, _dst, tns in executed_hops(executed, n)}
    for (j, t, src), tns in hop_t.items():
        prev = hop_t.get((j, t, src - 1))
        if src > 1 and prev is not None and prev > tns:
            order.append(f"hop of w{src} for stage {j} step {t} completed before the hop of w{src - 1}")
    return {"boundaries": len(per), "max_sends": max(counts), "min_sends": min(counts),
            "mean_sends": sum(counts) / len(counts), "max_sends_or_receives_per_worker": max_per_worker,
            "chain_order_violations": order}
