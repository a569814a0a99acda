"""Executed-version evidence on the device (ref engine.py:92-94 trace, :218-238 consistency check).

Trace-mode trainers tag every theta slot with the version of the data it holds (tags are written by
whoever writes the slot: set_params, the fused update, a parameter pull, a ZeRO-CDP state copy) and
record the tag found in the slot around every parameter read: forward reads (conv / BN / LayerNorm /
linear), backward reads (data-gradient GEMMs, BN / LayerNorm backward), the update's read of theta_t and
the slot it writes.  Checked bit-exactly against the rule table: forward AND backward reads of worker i
on stage j at step t see `rule.version_read(i, j, t)` (a backward reuses its forward's version, SURVEY
§4), before and after the access; the update reads t and writes t + 1.  The stage-level forward trace
(t, i, j, v) then passes the reference's `schedule_consistency_check` against the plan's timeline.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MB = 4


def _expected(rule, i, j, t):
    return t if rule is None else rule.version_read(i, j, t)


def _check_records(recs, world, rule, stage_of_unit, steps, n_units, backward_units):
    """Every record vs the rule; coverage of forward / backward / update records per (t, rank, unit)."""
    seen = set()
    for r in recs:
        t, rank, unit, kind, phase, slot, v = (int(r[k]) for k in r.dtype.names)
        i, j = rank + 1, int(stage_of_unit[unit - 1])
        if kind in (0, 1):
            want = _expected(rule, i, j, t)
        elif kind == 2:
            want = t
            assert rank == world - 1, "only the last worker updates"
        else:
            want = t + 1
            assert rank == world - 1
        assert v == want, dict(t=t, rank=rank, unit=unit, kind=kind, phase=phase, slot=slot, version=v, want=want)
        assert slot == (want & 1), (t, rank, unit, kind, slot, want)
        seen.add((t, rank, unit, kind, phase))
    for t in range(1, steps + 1):
        for rank in range(world):
            for u in range(1, n_units + 1):
                for ph in (0, 1):
                    assert (t, rank, u, 0, ph) in seen, ("forward", t, rank, u)
                    if u in backward_units:
                        assert (t, rank, u, 1, ph) in seen, ("backward", t, rank, u)
        for u in range(1, n_units + 1):
            assert (t, world - 1, u, 2, 0) in seen and (t, world - 1, u, 3, 1) in seen, ("update", t, u)


def _stage_trace(recs, stage_of_unit):
    return sorted({(int(r["t"]), int(r["rank"]) + 1, int(stage_of_unit[int(r["unit"]) - 1]), int(r["version"]))
                   for r in recs if r["kind"] == 0})


def _consistency(world, rule_name, steps, trace):
    from paper_2403_08837_b200 import ParallelismConfig, Scheme, build_cdp_timeline, build_dp_timeline
    from paper_2403_08837_b200.training import schedule_consistency_check

    if rule_name is None:
        tl = build_dp_timeline(ParallelismConfig(Scheme.MULTI_GPU_DP, world, 1, steps))
    else:
        tl = build_cdp_timeline(ParallelismConfig(Scheme.MULTI_GPU_CDP, world, 1, steps), rule_name)
    ok, bad = schedule_consistency_check(tl, trace)
    assert ok, bad
    # the device trace covers every forward task of the plan
    fwd = {(t.training_step, t.micro_batch, t.stage) for t in tl.tasks if t.kind.name == "FORWARD"}
    assert fwd == {(t, i, j) for t, i, j, _ in trace}


@pytest.mark.parametrize("world,rule_name,zero", [(1, None, False), (2, None, False), (2, "cdp-v1", False),
                                                  (2, "cdp-v2", False), (3, "cdp-v2", False), (4, "cdp-v1", False),
                                                  (4, "cdp-v2", False), (3, "cdp-v2", True)])
def test_resnet_executed_versions(cuda, world, rule_name, zero):
    from oracle.resnet_torch import init_flat
    from paper_2403_08837_b200.resnet import DeviceResNet, synthetic_cifar
    from paper_2403_08837_b200.rules import rule_by_name

    rule = rule_by_name(rule_name, world) if rule_name else None
    W, D, hw = (64, 128), (1, 1), 16
    x, y = synthetic_cifar(world * MB * 2, 0, hw=hw)
    init = init_flat(W, D, seed=0)
    steps = 4
    tr = [DeviceResNet(W, D, MB, world, r, rule, "bf16", 0.9, inputs=x, labels=y, image_hw=hw, zero=zero,
                       trace=True) for r in range(world)]
    regions = [t.region() for t in tr]
    for t in tr:
        t.set_params(init, -1)
        t.connect(regions)
    for k in range(steps):
        perm = np.random.default_rng([3, k]).permutation(len(x))
        for r, t in enumerate(tr):
            t.step(perm[r * MB:(r + 1) * MB], 0.05)
    for t in tr:
        t.zero_drain()
    for t in tr:
        t.sync()
        assert t.ring_error() == 0
    recs = np.concatenate([t.access_trace() for t in tr])
    stage = tr[0].stage
    kinds = [k for k, _, _ in tr[0].specs]
    n_units = len(kinds)
    # the stem convolution's weight has no data gradient (its only backward access is the hop)
    backward_units = {u for u in range(1, n_units + 1) if u != 1}
    for t in tr:
        t.close()
    _check_records(recs, world, rule, stage, steps, n_units, backward_units)
    _consistency(world, rule_name, steps, _stage_trace(recs, stage))


@pytest.mark.parametrize("world,rule_name,dtype", [(1, None, "bf16"), (2, "cdp-v2", "bf16"), (3, "cdp-v1", "bf16"),
                                                   (3, "cdp-v2", "bf16"), (2, "cdp-v2", "fp32"), (3, "cdp-v1", "fp32")])
def test_vit_executed_versions(cuda, world, rule_name, dtype):
    from paper_2403_08837_b200.rules import rule_by_name
    from paper_2403_08837_b200.vit import DeviceVit, vit_init

    rule = rule_by_name(rule_name, world) if rule_name else None
    cfg = dict(image=32, patch=16, dim=128, depth=2, heads=2, mlp=256, classes=10)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(world * MB * 2, 32, 32, 3)).astype(np.float32)
    y = rng.integers(0, 10, size=len(x)).astype(np.int32)
    steps = 4
    tr = [DeviceVit(cfg, MB, world, r, rule, 0.9, inputs=x, labels=y, trace=True, dtype=dtype) for r in range(world)]
    regions = [t.region() for t in tr]
    init = vit_init(cfg, 0)
    for t in tr:
        t.set_params(init, -1)
        t.connect(regions)
    for k in range(steps):
        perm = np.random.default_rng([4, k]).permutation(len(x))
        for r, t in enumerate(tr):
            t.step(perm[r * MB:(r + 1) * MB], 0.05)
    for t in tr:
        t.sync()
        assert t.ring_error() == 0
    recs = np.concatenate([t.access_trace() for t in tr])
    stage = tr[0].stage
    names = [n for n, _, _ in tr[0].units]
    n_units = len(names)
    # cls / pos / patch weights have no backward read (their gradients need no parameter)
    backward_units = {u + 1 for u, n in enumerate(names) if n not in ("cls", "pos", "patch")}
    for t in tr:
        t.close()
    _check_records(recs, world, rule, stage, steps, n_units, backward_units)
    _consistency(world, rule_name, steps, _stage_trace(recs, stage))
