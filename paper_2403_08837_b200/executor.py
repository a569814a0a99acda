"""Compile a reference-parity Timeline into the device step plan.

The cyclic step scheduler has two halves: this planner (host, pure Python,
unit-tested on CPU) and the native executor in
`csrc/mlp_trainer.cu` that captures the plan into CUDA graphs.

Input: the Timeline of the configured scheme (`schedule.build_cdp_timeline`
/ `build_dp_timeline`, bit-exact with ref `schedule.py:178-257`).
Output (`StepPlan`), for one training step in steady state:

* `ops`   one row per F/B task in timeline order (start, worker):
          [kind(0=F,1=B), worker i, stage j, fresh, rec_in, rec_out, hop, 0]
          - fresh: the rule's table (ref `rules.py:45-51`); the executor reads
            stage j from version slot t mod 2 (fresh) or (t-1) mod 2 (stale);
          - rec_in / rec_out: activation-record slots (the stage-j input of
            micro-batch i lives from its producer F(i, j-1) to B(i, j));
          - hop: role of B(i, j) in the gradient chain w1 -> ... -> wN
            (ref `comm.py:37-67`, ascending-i order of `engine.py:96-101`):
            0 first, 1 middle, 2 last (fused update), 3 only (N = 1);
* `deps`  cross-worker edges (before_op, after_op): the ring hop
          B(i-1, j) -> B(i, j) and activation-slot reuse B(i, j) -> producer
          of the next record in that slot;
* `slots` activation-record slots per stage, so peak activation memory is
          the interval-colouring of the plan, not N records per stage.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .profiles import CostWeights, ParallelismConfig, Scheme
from .rules import UpdateRule
from .schedule import TaskKind, build_cdp_timeline, build_dp_timeline

OP_FIELDS = 8
OP_F, OP_B, OP_PULL = 0, 1, 2
HOP_FIRST, HOP_MID, HOP_LAST, HOP_ONLY, HOP_GRAD = 0, 1, 2, 3, 4


@dataclass
class StepPlan:
    n_stages: int
    n_workers: int
    ops: np.ndarray      # int32 [n_ops, OP_FIELDS]
    deps: np.ndarray     # int32 [n_deps, 2]
    slots: np.ndarray    # int32 [n_stages + 1], slots[j] for stage j (index 0 unused)
    fresh: np.ndarray    # uint8 [n_workers, n_stages]

    def trace(self, step: int) -> list:
        """(t, i, j, version) reads of one step, ascending i then j (ref engine.py:92-94)."""
        out = []
        for i in range(1, self.n_workers + 1):
            for j in range(1, self.n_stages + 1):
                out.append((step, i, j, step if self.fresh[i - 1, j - 1] else step - 1))
        return out


def _template_tasks(n_stages: int, n_workers: int, rule: UpdateRule | None, weights: CostWeights):
    """(start, worker, kind, stage) for one steady step of the plan."""
    if n_stages == n_workers:
        scheme = Scheme.SINGLE_GPU_DP if rule is None else Scheme.SINGLE_GPU_CDP
        cfg = ParallelismConfig(scheme, n_workers, 1, 2, weights)
        tl = build_dp_timeline(cfg) if rule is None else build_cdp_timeline(cfg, rule)
        return [(t.start, t.micro_batch, 0 if t.kind is TaskKind.FORWARD else 1, t.stage)
                for t in tl.tasks if t.training_step == 2]
    if rule is not None:
        raise ValueError("a cyclic rule ties stages to micro-batches (n x n table)")
    fc, bc = weights.forward_cost, weights.backward_cost
    out = []
    for i in range(1, n_workers + 1):
        for j in range(1, n_stages + 1):
            out.append(((j - 1) * fc + 1, i, 0, j))
            out.append((n_stages * fc + (n_stages - j) * bc + 1, i, 1, j))
    return out


def layer_stages(n_layers: int, n_stages: int) -> list:
    """Contiguous, balanced assignment of layers to stages (1-based stage per layer)."""
    if not 1 <= n_stages <= n_layers:
        raise ValueError("need 1 <= stages <= layers")
    base, extra = divmod(n_layers, n_stages)
    out = []
    for s in range(1, n_stages + 1):
        out += [s] * (base + (1 if s <= extra else 0))
    return out


def _check_stage_map(layer_stage, n_stages):
    if list(layer_stage) != sorted(layer_stage) or set(layer_stage) != set(range(1, n_stages + 1)):
        raise ValueError("layer_stage must map layers onto stages 1..n contiguously")


def compile_step_plan(n_stages: int, n_workers: int, rule: UpdateRule | None = None,
                      weights: CostWeights = CostWeights(), grad_only: bool = False,
                      layer_stage=None) -> StepPlan:
    """Single-GPU plan; with `layer_stage` a stage task expands into its layers
    (F ascending, B descending), all reading the stage's version."""
    if layer_stage is None:
        layer_stage = list(range(1, n_stages + 1))
    _check_stage_map(layer_stage, n_stages)
    n_layers = len(layer_stage)
    layers_of = {s: [l for l in range(1, n_layers + 1) if layer_stage[l - 1] == s] for s in range(1, n_stages + 1)}
    if rule is not None:
        if rule.n != n_workers:
            raise ValueError("rule size does not match task")
        rule.check_feasible()
    tasks = sorted(_template_tasks(n_stages, n_workers, rule, weights), key=lambda x: (x[0], x[1], x[2]))
    fresh = np.ones((n_workers, n_stages), dtype=np.uint8)
    if rule is not None:
        fresh[:] = np.array(rule.fresh, dtype=np.uint8)

    ops, deps = [], []
    index = {}
    free = {l: [] for l in range(1, n_layers + 1)}     # free record slots per layer input
    count = {l: 0 for l in range(1, n_layers + 1)}
    last_user = {}                                     # (l, slot) -> op that released it
    holder = {}                                        # (i, l) -> slot of record (i, l)

    def acquire(l: int, producer_op: int) -> int:
        if free[l]:
            s = free[l].pop(0)
            rel = last_user.get((l, s))
            if rel is not None:
                deps.append((rel, producer_op))
        else:
            s = count[l]
            count[l] += 1
        return s

    for _start, i, kind, stage in tasks:
        f = int(fresh[i - 1, stage - 1])
        seq = layers_of[stage] if kind == 0 else layers_of[stage][::-1]
        for l in seq:
            o = len(ops)
            row = [kind, i, l, f, 0, 0, 0, 0]
            if kind == 0:
                if l == 1:
                    holder[(i, 1)] = acquire(1, o)
                row[4] = holder[(i, l)]
                if l < n_layers:
                    holder[(i, l + 1)] = acquire(l + 1, o)
                    row[5] = holder[(i, l + 1)]
            else:
                row[4] = holder[(i, l)]
                if grad_only:
                    row[6] = HOP_GRAD
                elif n_workers == 1:
                    row[6] = HOP_ONLY
                else:
                    row[6] = HOP_FIRST if i == 1 else (HOP_LAST if i == n_workers else HOP_MID)
                if i > 1 and not grad_only:
                    deps.append((index[(1, i - 1, l)], o))
                s = holder.pop((i, l))
                free[l].append(s)
                last_user[(l, s)] = o
            index[(kind, i, l)] = o
            ops.append(row)

    deps = sorted(set(deps))
    for a, b in deps:
        assert a < b, "plan edges must point forward"
    slots = np.zeros(n_layers + 1, dtype=np.int32)
    for l in range(1, n_layers + 1):
        slots[l] = max(count[l], 1)
    return StepPlan(
        n_stages, n_workers,
        np.asarray(ops, dtype=np.int32).reshape(-1, OP_FIELDS),
        np.asarray(deps, dtype=np.int32).reshape(-1, 2),
        slots, fresh,
    )


def record_bytes(plan: StepPlan, dims, micro_batch: int, elem_bytes: int) -> int:
    """Activation bytes the executor allocates for `plan` (record l = input of layer l)."""
    pad = lambda c: (c + 15) // 16 * 16
    return int(sum(int(plan.slots[l]) * micro_batch * pad(dims[l - 1]) * elem_bytes
                   for l in range(1, len(plan.slots))))


def compile_rank_plan(n_workers: int, rank: int, rule: UpdateRule | None = None, layer_stage=None,
                      allreduce: bool = False) -> np.ndarray:
    """Op list of one rank in multi-GPU CDP / DP (worker i = rank + 1 on its own GPU).

    Per step: [pull(j)] F(i, j) for j = 1..N, then B(i, j) for j = N..1.  The
    pull fetches, from the updater rank N-1, the version of stage j this
    worker reads (t if fresh else t-1, ref rules.py:48-51) right before the
    forward that reads it; the updater itself never pulls.  Every version is
    therefore pulled exactly once per reader (fresh readers at step v, stale
    readers at step v+1), which is what the updater's overwrite guard counts.
    Record slots are all 0: one micro-batch per GPU holds one record per layer.
    With `layer_stage`, pulls and hops run per layer (the per-layer delayed
    gradient path) while versions follow the layer's stage.
    """
    n = n_workers
    i = rank + 1
    if not 0 <= rank < n:
        raise ValueError("rank out of range")
    if layer_stage is None:
        layer_stage = list(range(1, n + 1))
    _check_stage_map(layer_stage, n)
    n_layers = len(layer_stage)
    if rule is not None:
        if rule.n != n:
            raise ValueError("rule size does not match the number of ranks")
        rule.check_feasible()
    fresh = (lambda l: 1) if rule is None else (lambda l: int(rule.reads_fresh(i, layer_stage[l - 1])))
    hop = HOP_ONLY if n == 1 else HOP_FIRST if i == 1 else HOP_LAST if i == n else HOP_MID
    if allreduce:  # DP baseline: own gradient only; the collective + update run after the step
        if rule is not None:
            raise ValueError("the all-reduce baseline is synchronous DP (rule None)")
        hop = HOP_GRAD
    ops = []
    for l in range(1, n_layers + 1):
        if i != n and not allreduce:
            ops.append([OP_PULL, i, l, fresh(l), 0, 0, 0, 0])
        ops.append([OP_F, i, l, fresh(l), 0, 0, 0, 0])
    for l in range(n_layers, 0, -1):
        ops.append([OP_B, i, l, fresh(l), 0, 0, hop, 0])
    return np.asarray(ops, dtype=np.int32)


@dataclass
class SegmentPlan:
    """Single-GPU plan over model segments (one worker = one micro-batch, all on one GPU).

    ops     int32 [n_ops, 3]: (kind 0=F / 1=B, worker i, stage j) in timeline order;
    slot    int32 [n_workers, n_segments]: activation-record slot of (i, segment) in its pool;
    pools   int32 [n_pools]: slots per record pool (the interval colouring's width);
    live    int32 [n_ops + 1, n_pools]: records live after each op (index 0 = before the step);
    fresh   uint8 [n_workers, n_stages]: the rule table (all ones for DP)."""

    ops: np.ndarray
    slot: np.ndarray
    pools: np.ndarray
    live: np.ndarray
    fresh: np.ndarray

    def peak_bytes(self, record_bytes) -> int:
        """High-water mark of live record bytes over the step (time-resolved, not pools x bytes)."""
        return int((self.live.astype(np.int64) @ np.asarray(record_bytes, dtype=np.int64)).max())


def segment_partition(seg_cost, n_stages: int) -> np.ndarray:
    """Contiguous split of segments into `n_stages` non-empty stages minimising the largest stage
    cost (exact DP; ties keep earlier boundaries).  Returns the 1-based stage of each segment."""
    cost = np.asarray(seg_cost, dtype=np.float64)
    S = len(cost)
    if not 1 <= n_stages <= S:
        raise ValueError("need 1 <= stages <= segments")
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    INF = float("inf")
    best = np.full((n_stages + 1, S + 1), INF)
    cut = np.zeros((n_stages + 1, S + 1), dtype=np.int64)
    best[0, 0] = 0.0
    for k in range(1, n_stages + 1):
        for e in range(k, S + 1):
            for b in range(k - 1, e):
                v = max(best[k - 1, b], cum[e] - cum[b])
                if v < best[k, e]:
                    best[k, e], cut[k, e] = v, b
    stage = np.zeros(S, dtype=np.int32)
    e = S
    for k in range(n_stages, 0, -1):
        b = int(cut[k, e])
        stage[b:e] = k
        e = b
    return stage


def compile_segment_plan(n_workers: int, seg_stage, seg_pool, rule: UpdateRule | None = None,
                         weights: CostWeights = CostWeights()) -> SegmentPlan:
    """Cyclic (rule) or lockstep DP (rule None) single-GPU plan from the reference Timeline
    (SINGLE_GPU_CDP / SINGLE_GPU_DP, ref schedule.py:178-257) expanded onto segments.

    The record of (worker i, segment s) holds s's input and what B(i, s) reads: it is acquired by
    the forward that writes that input (F of segment s-1; segment 0 by its own forward) and
    released after B(i, s).  Slots are coloured greedily in timeline order (lowest free slot), which
    for these interval graphs uses exactly the maximum number of simultaneously live records — the
    (N+1)/2 vs N micro-batches of ref costs.py:111-115 when the segments are homogeneous."""
    n = n_workers
    seg_stage = [int(s) for s in seg_stage]
    seg_pool = [int(p) for p in seg_pool]
    S = len(seg_stage)
    if len(seg_pool) != S:
        raise ValueError("seg_pool must name a pool per segment")
    _check_stage_map(seg_stage, n)
    if rule is not None:
        if rule.n != n:
            raise ValueError("rule size does not match the number of workers")
        rule.check_feasible()
    tasks = sorted(_template_tasks(n, n, rule, weights), key=lambda x: (x[0], x[1], x[2]))
    fresh = np.ones((n, n), dtype=np.uint8)
    if rule is not None:
        fresh[:] = np.array(rule.fresh, dtype=np.uint8)
    n_pools = max(seg_pool) + 1
    free = [[] for _ in range(n_pools)]
    count = [0] * n_pools
    live = [0] * n_pools
    slot = -np.ones((n, S), dtype=np.int32)
    held = set()
    curve = [list(live)]
    ops = []

    def acquire(i, s):
        k = seg_pool[s]
        if free[k]:
            free[k].sort()
            v = free[k].pop(0)
        else:
            v = count[k]
            count[k] += 1
        if slot[i - 1, s] not in (-1, v):
            raise AssertionError("a record must keep its slot from step to step (periodic plan)")
        slot[i - 1, s] = v
        held.add((i, s))
        live[k] += 1

    def release(i, s):
        k = seg_pool[s]
        held.remove((i, s))
        free[k].append(int(slot[i - 1, s]))
        live[k] -= 1

    segs_of = {j: [s for s in range(S) if seg_stage[s] == j] for j in range(1, n + 1)}
    for _start, i, kind, j in tasks:
        ops.append((kind, i, j))
        if kind == 0:
            for s in segs_of[j]:
                if s == 0:
                    acquire(i, 0)
                if s + 1 < S:
                    acquire(i, s + 1)
        else:
            for s in segs_of[j][::-1]:
                release(i, s)
        curve.append(list(live))
    if held:
        raise AssertionError("every record must be released by the end of the step")
    return SegmentPlan(np.asarray(ops, dtype=np.int32).reshape(-1, 3), slot,
                       np.asarray([max(c, 1) for c in count], dtype=np.int32),
                       np.asarray(curve, dtype=np.int32), fresh)


def plan_live_peak(plan: StepPlan, dims, micro_batch: int, elem_bytes: int) -> dict:
    """Peak of the LIVE activation records over the plan's op order (the order the executor issues them):
    record (i, l) - the input of layer l for micro-batch i - is live from the forward that produces it to
    the backward of layer l.  The time-resolved quantity the reference's (N+1)/2-vs-N record count is
    about (ref costs.py:111-115); the allocation (`record_bytes`) keeps per-layer slots for the whole step,
    so with unequal layer widths its ratio is larger."""
    pad = lambda c: (c + 15) // 16 * 16
    size = {l: micro_batch * pad(dims[l - 1]) * elem_bytes for l in range(1, len(dims))}
    live, peak_b, peak_n, cur_b, cur_n = set(), 0, 0, 0, 0
    n_layers = len(dims) - 1
    for row in plan.ops:
        kind, i, l = int(row[0]), int(row[1]), int(row[2])
        if kind == OP_F:
            for rec in ([(i, 1)] if l == 1 else []) + ([(i, l + 1)] if l < n_layers else []):
                if rec not in live:
                    live.add(rec)
                    cur_b += size[rec[1]]
                    cur_n += 1
        elif kind == OP_B and (i, l) in live:
            live.discard((i, l))
            cur_b -= size[l]
            cur_n -= 1
        peak_b, peak_n = max(peak_b, cur_b), max(peak_n, cur_n)
    return {"peak_live_bytes": peak_b, "peak_live_records": peak_n}
