"""ZeRO-CDP state passing: the device protocol derived from the reference plan.

Reference: `comm.schedule_zero_transfers` (ref `comm.py:93-144`) over the
cyclic ZeRO placement `build_zero_timeline(cyclic=True)` (ref
`schedule.py:433-472`, CDP-v2 placement): exactly one worker uses a stage per
time step; the stage's model state hops point-to-point from its holder to
its next user and is freed at the source.

Device protocol (csrc/resnet_trainer.cu, ZeRO mode).  For every stage s the
uses (F or B tasks of any worker) are totally ordered by start time; the
schedule is periodic with 2N uses per step (N forwards + N backwards).  A use
of kind k by worker i in training step t has the global use index

    u = base[s][k][i] + (t - 1) * 2N

and its predecessor (the previous use of stage s) is the use of worker
prev[s][k][i] in step t + dstep[s][k][i].  Before its first access to a
tensor of stage s the user waits until the predecessor's rank has published
`zdone[tensor] >= u - 1`, copies the tensor's state (both version slots of
theta and the momentum) from that rank's HBM, and after its last access
publishes `zdone[tensor] = u`.  Uses whose predecessor would lie before step
1 read the initial state every rank holds.  This module computes base / prev /
dstep from the reference-parity plan and re-derives the transfer events from
them (tests/test_zero_plan.py compares both with `schedule_zero_transfers`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .comm import schedule_zero_transfers
from .profiles import ParallelismConfig, Scheme, make_homogeneous_profile
from .schedule import TaskKind, build_zero_timeline

KINDS = (TaskKind.FORWARD, TaskKind.BACKWARD)


@dataclass(frozen=True)
class ZeroPlan:
    n: int
    base: np.ndarray    # [n_stages][2][n] int32: global use index of (kind, worker i) in step 1
    prev: np.ndarray    # [n_stages][2][n] int32: 0-based rank of the previous use's worker
    dstep: np.ndarray   # [n_stages][2][n] int32: step offset of the previous use (-1, 0 or +1)
    uses_per_step: int  # 2N

    def table(self) -> np.ndarray:
        """[n_stages][2][n][3] int32 (base, prev rank, dstep) for the C ABI."""
        return np.ascontiguousarray(np.stack([self.base, self.prev, self.dstep], axis=-1).astype(np.int32))


def _worker(device: str) -> int:
    return int(device[1:])


def zero_plan(n: int, steps: int = 6) -> ZeroPlan:
    """Derive the periodic use order of every stage from the reference-parity ZeRO-CDP timeline."""
    if n < 1:
        raise ValueError("n must be >= 1")
    cfg = ParallelismConfig(scheme=Scheme.ZERO_CDP, n=n, training_steps=max(steps, 4))
    tl = build_zero_timeline(cfg, make_homogeneous_profile(n, n, n, 1), cyclic=True)
    per = 2 * n
    base = np.zeros((n, 2, n), dtype=np.int64)
    prev = np.zeros((n, 2, n), dtype=np.int64)
    dstep = np.zeros((n, 2, n), dtype=np.int64)
    t_ref = 3  # a steady-state step
    for s in range(1, n + 1):
        uses = sorted((t for t in tl.tasks if t.stage == s), key=lambda t: t.start)
        index = {(t.kind, t.micro_batch, t.training_step): k for k, t in enumerate(uses)}
        for ki, kind in enumerate(KINDS):
            for i in range(1, n + 1):
                u = index[(kind, i, t_ref)]
                u2 = index[(kind, i, t_ref + 1)]
                if u2 - u != per:
                    raise AssertionError("ZeRO-CDP use order is not periodic")
                base[s - 1, ki, i - 1] = u - (t_ref - 1) * per
                p = uses[u - 1]
                prev[s - 1, ki, i - 1] = _worker(p.device) - 1
                dstep[s - 1, ki, i - 1] = p.training_step - t_ref
                if p.training_step > t_ref:
                    # a use may follow a FORWARD of the next step (never a backward): the device's
                    # end-of-run drain publishes exactly those forwards (drain_units)
                    if p.kind is not TaskKind.FORWARD or kind is not TaskKind.BACKWARD:
                        raise AssertionError("unexpected next-step predecessor in the ZeRO-CDP plan")
                    pp = uses[u - 2]
                    if pp.training_step > t_ref + 1 or (pp.training_step == t_ref + 1 and pp.kind is TaskKind.BACKWARD):
                        raise AssertionError("a drained forward must only depend on earlier steps")
    # make every index non-negative (the device compares unsigned step counters)
    base -= base.min()
    return ZeroPlan(n, base.astype(np.int32), prev.astype(np.int32), dstep.astype(np.int32), per)


def drain_units(plan: ZeroPlan, rank: int) -> list:
    """Stages (1-based) whose next-step forward on `rank` is the predecessor of a backward of the current
    step on another rank: the end-of-run drain publishes exactly these uses."""
    out = []
    for s in range(plan.n):
        if any(int(plan.prev[s, 1, j]) == rank and int(plan.dstep[s, 1, j]) == 1 for j in range(plan.n)):
            out.append(s + 1)
    return out


def transfers(plan: ZeroPlan, steps: int) -> list:
    """(step, kind, stage, src rank, dst rank) of every state copy the device protocol performs,
    in use order per stage - the event list `schedule_zero_transfers` emits (src != dst)."""
    out = []
    n = plan.n
    for s in range(n):
        ev = []
        for t in range(1, steps + 1):
            for ki in range(2):
                for i in range(n):
                    pt = t + int(plan.dstep[s, ki, i])
                    u = int(plan.base[s, ki, i]) + (t - 1) * plan.uses_per_step
                    src = int(plan.prev[s, ki, i])
                    if pt >= 1 and src != i:
                        ev.append((u, t, ki, s + 1, src, i))
        out.extend(sorted(ev))
    return [e[1:] for e in out]


def reference_transfers(n: int, steps: int) -> list:
    """The reference plan's STATE_TRANSFER events as (step of the receiving use, kind, stage, src, dst)."""
    cfg = ParallelismConfig(scheme=Scheme.ZERO_CDP, n=n, training_steps=steps)
    prof = make_homogeneous_profile(n, n, n, 1)
    tl = schedule_zero_transfers(build_zero_timeline(cfg, prof, cyclic=True), True, prof)
    user = {(t.start, t.stage): t for t in tl.tasks}
    out = []
    for e in tl.comm_events:
        if e.kind.value != "state-transfer":
            continue
        t = user[(e.boundary + 1, e.stage)]
        out.append((t.start, t.training_step, KINDS.index(t.kind), e.stage, _worker(e.src) - 1, _worker(e.dst) - 1))
    return [o[1:] for o in sorted(out, key=lambda o: (o[3], o[0]))]


def state_bytes_per_step(plan: ZeroPlan, stage_params, rank: int, momentum: bool = True) -> int:
    """Bytes one rank receives per steady step: both theta slots (+ momentum) of every received stage use."""
    per_param = 4 * (2 + (1 if momentum else 0))
    total = 0
    for s in range(plan.n):
        for ki in range(2):
            if int(plan.prev[s, ki, rank]) != rank:
                total += per_param * int(stage_params[s])
    return total



def frame_drain_plan(n: int) -> list:
    """End-of-run drain of ZeRO-CDP state frames (csrc/resnet_trainer.cu), per rank.

    A rank keeps the state of stage s in frame (s - 1) & 1 and reuses a frame once the previous
    occupant's successor has copied it out.  In the CDP-v2 ZeRO placement the last ranks' late backward
    windows hand their state to NEXT-step forwards of earlier ranks (N = 4: w4's B2 -> w1's F4 of step
    t + 1), so at the end of a run those forwards' state copies must still happen: the drain of rank r
    copies stage s's state for its next-step forward, for every s in the returned list, in order (the
    closure: forwards whose copy a frame reuse waits for, their own frame reuses, their predecessors).
    Each entry is (stage s (1-based), previous occupant stage (0-based, -1: none), kind of its last
    use, that use's step offset and its successor's step offset from it): the frame wait before the
    copy, relative to the drain's step (the next, unlaunched one).  A drained run cannot continue."""
    cfg = ParallelismConfig(scheme=Scheme.ZERO_CDP, n=n, training_steps=8)
    tl = build_zero_timeline(cfg, make_homogeneous_profile(n, n, n, 1), cyclic=True)
    tasks = [t for t in tl.tasks if t.kind in KINDS]
    T = 4  # a steady last step; offsets are relative to T + 1
    succ, pred = {}, {}
    for s in range(1, n + 1):
        uses = sorted((t for t in tasks if t.stage == s), key=lambda t: t.start)
        for a, b in zip(uses, uses[1:]):
            succ[id(a)], pred[id(b)] = b, a
    devs = [f"w{r + 1}" for r in range(n)]
    seqs = {d: sorted((t for t in tasks if t.device == d), key=lambda t: t.start) for d in devs}

    def windows(d):
        wins = []
        for t in seqs[d]:
            if wins and wins[-1][-1].stage == t.stage:
                wins[-1].append(t)
            else:
                wins.append([t])
        return wins

    drained = set()

    def executed(t):  # ran in steps <= T, or in the drain (F1 of T + 1 is a no-copy publish)
        return t.training_step <= T or id(t) in drained or (
            t.training_step == T + 1 and t.kind is TaskKind.FORWARD and t.stage == 1)

    waits = {}
    changed = True
    while changed:
        changed = False
        waits = {}
        for d in devs:
            last_in_frame = {}
            for w in windows(d):
                if not executed(w[0]):
                    continue
                f = (w[0].stage - 1) & 1
                occ = last_in_frame.get(f)
                p = pred.get(id(w[0]))
                copies = p is not None and p.device != d
                if copies and id(w[0]) in drained:
                    if occ is None:
                        waits[id(w[0])] = (-1, 0, 0, 0)
                    else:
                        lu = [t for t in occ if executed(t)][-1]
                        sc = succ[id(lu)]
                        waits[id(w[0])] = (lu.stage - 1, KINDS.index(lu.kind), lu.training_step - (T + 1),
                                           sc.training_step - lu.training_step)
                if occ is not None and copies:
                    lu = [t for t in occ if executed(t)][-1]
                    sc = succ.get(id(lu))
                    if sc is not None and not executed(sc):
                        if sc.kind is not TaskKind.FORWARD or sc.training_step != T + 1:
                            raise AssertionError("ZeRO-CDP frames: a frame reuse waits on an undrainable use")
                        drained.add(id(sc))
                        changed = True
                last_in_frame[f] = w
        for i in list(drained):
            t = next(x for x in tasks if id(x) == i)
            p = pred[i]
            if not executed(p):
                if p.kind is not TaskKind.FORWARD or p.training_step != T + 1:
                    raise AssertionError("ZeRO-CDP frames: a drained forward has an undrainable predecessor")
                drained.add(id(p))
                changed = True
    out = []
    for r, d in enumerate(devs):
        rows = sorted(((t.stage,) + waits[id(t)] for t in tasks if id(t) in drained and t.device == d))
        out.append(rows)
    return out
