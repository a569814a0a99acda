"""Step-plan compiler (host half of the cyclic scheduler), CPU only."""

import numpy as np
import pytest

from paper_2403_08837_b200.executor import HOP_FIRST, HOP_LAST, HOP_MID, HOP_ONLY, compile_step_plan, record_bytes
from paper_2403_08837_b200.rules import generic_rule, max_delay_rule, min_delay_rule


def _simulate_slots(plan):
    """Replay ops in order; every record read must be the one written into that slot."""
    owner = {}
    for o, (kind, i, j, fresh, rin, rout, hop, _) in enumerate(plan.ops):
        if kind == 0:
            if j == 1:
                owner[(1, rin)] = (i, o)
            assert owner[(j, rin)][0] == i, "forward reads another micro-batch's record"
            if j < plan.n_stages:
                owner[(j + 1, rout)] = (i, o)
        else:
            assert owner[(j, rin)][0] == i, "backward reads another micro-batch's record"


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("rule", ["dp", "v1", "v2"])
def test_plan_structure(n, rule):
    r = None if rule == "dp" else (max_delay_rule(n) if rule == "v1" else min_delay_rule(n))
    plan = compile_step_plan(n, n, r)
    assert plan.ops.shape == (2 * n * n, 8)
    assert all(a < b for a, b in plan.deps)
    _simulate_slots(plan)
    # every B task has the hop role of its position in the ascending ring
    for kind, i, j, fresh, *_rest in plan.ops:
        if kind == 1:
            hop = _rest[2]
            want = HOP_ONLY if n == 1 else HOP_FIRST if i == 1 else HOP_LAST if i == n else HOP_MID
            assert hop == want
        if r is not None:
            assert fresh == int(r.reads_fresh(i, j))
        else:
            assert fresh == 1
    # ring edges B(i-1,j) -> B(i,j)
    idx = {(int(k), int(i), int(j)): o for o, (k, i, j, *_x) in enumerate(plan.ops)}
    dset = {tuple(map(int, d)) for d in plan.deps}
    for j in range(1, n + 1):
        for i in range(2, n + 1):
            assert (idx[(1, i - 1, j)], idx[(1, i, j)]) in dset


@pytest.mark.parametrize("n", [2, 3, 4, 6, 8])
def test_cdp_holds_triangular_records_dp_holds_square(n):
    """CDP keeps N-j+1 records of stage j alive (total N(N+1)/2), DP keeps N per stage
    (ref costs.py:111-115: (N+1)/2 vs N micro-batches of activations)."""
    cdp = compile_step_plan(n, n, min_delay_rule(n))
    dp = compile_step_plan(n, n, None)
    assert list(cdp.slots[1:]) == [n - j + 1 for j in range(1, n + 1)]
    assert list(dp.slots[1:]) == [n] * n
    assert int(cdp.slots.sum()) == n * (n + 1) // 2
    dims = (64,) * (n + 1)
    assert record_bytes(cdp, dims, 32, 4) * 2 * n == record_bytes(dp, dims, 32, 4) * (n + 1)


def test_plan_generic_rule_and_errors():
    table = [[False, False, True], [False, True, True], [False, False, False]]
    plan = compile_step_plan(3, 3, generic_rule(table))
    assert plan.fresh.tolist() == [[0, 0, 1], [0, 1, 1], [0, 0, 0]]
    with pytest.raises(ValueError):
        compile_step_plan(3, 4, min_delay_rule(4))
    with pytest.raises(ValueError):
        compile_step_plan(4, 4, min_delay_rule(3))


def test_trace_matches_rule():
    plan = compile_step_plan(4, 4, min_delay_rule(4))
    tr = plan.trace(7)
    assert (7, 2, 3, 7) in tr and (7, 2, 2, 6) in tr and len(tr) == 16


def test_layer_stage_grouping():
    from paper_2403_08837_b200.executor import compile_rank_plan, layer_stages

    assert layer_stages(8, 4) == [1, 1, 2, 2, 3, 3, 4, 4]
    assert layer_stages(7, 3) == [1, 1, 1, 2, 2, 3, 3]
    r = min_delay_rule(4)
    plan = compile_step_plan(4, 4, r, layer_stage=layer_stages(8, 4))
    assert plan.ops.shape == (2 * 4 * 8, 8)
    _simulate_slots_layers(plan, 8)
    for kind, i, l, fresh, *_x in plan.ops:
        assert fresh == int(r.reads_fresh(i, (l + 1) // 2))
    ops = compile_rank_plan(4, 1, r, layer_stages(8, 4))
    kinds = [tuple(o[:3]) for o in ops]
    assert kinds[:4] == [(2, 2, 1), (0, 2, 1), (2, 2, 2), (0, 2, 2)]
    assert kinds[-1] == (1, 2, 1)
    with pytest.raises(ValueError):
        compile_step_plan(4, 4, r, layer_stage=[1, 3, 2, 4])


def _simulate_slots_layers(plan, n_layers):
    owner = {}
    for kind, i, l, fresh, rin, rout, hop, _ in plan.ops:
        if kind == 0:
            if l == 1:
                owner[(1, rin)] = i
            assert owner[(l, rin)] == i
            if l < n_layers:
                owner[(l + 1, rout)] = i
        else:
            assert owner[(l, rin)] == i


def test_plan_live_record_peak_matches_reference_count():
    """Single-GPU CDP holds N(N+1)/2 live records at its peak against DP's N^2 (ref costs.py:111-115), over the
    op order the executor issues; with layer 1 much wider than the rest the byte ratio stays larger."""
    from paper_2403_08837_b200.executor import compile_step_plan, plan_live_peak
    from paper_2403_08837_b200.rules import rule_by_name

    for n in (2, 3, 4, 6):
        dims = [64] * (n + 1)
        dp = plan_live_peak(compile_step_plan(n, n, None), dims, 8, 2)
        assert dp["peak_live_records"] == n * n
        for r in ("cdp-v1", "cdp-v2"):
            cdp = plan_live_peak(compile_step_plan(n, n, rule_by_name(r, n)), dims, 8, 2)
            assert cdp["peak_live_records"] == n * (n + 1) // 2, (n, r)
    wide = [3072, 256, 256, 256, 10]
    cdp = plan_live_peak(compile_step_plan(4, 4, rule_by_name("cdp-v1", 4)), wide, 32, 2)
    dp = plan_live_peak(compile_step_plan(4, 4, None), wide, 32, 2)
    assert 0.8 < cdp["peak_live_bytes"] / dp["peak_live_bytes"] < 0.95
