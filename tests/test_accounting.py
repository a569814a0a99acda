"""Executed-schedule accounting (paper_2403_08837_b200/accounting.py) on CPU: an "execution" that follows
the plan exactly (each time step mapped to a device-time interval) must reproduce the plan's own
activation peak (ref costs.py:157-170 records) and the plan's gradient-hop balance (ref comm.py:37-67,
196-221) — the measured accounting is then fed device stamps in tests/test_gpu_accounting.py."""

import pytest

from paper_2403_08837_b200.accounting import activation_series_ns, executed_activation, executed_balance
from paper_2403_08837_b200.cli import _planned_peak
from paper_2403_08837_b200.comm import balance_report, schedule_cdp_ring_reduce
from paper_2403_08837_b200.profiles import ParallelismConfig, Scheme, make_homogeneous_profile
from paper_2403_08837_b200.rules import rule_by_name
from paper_2403_08837_b200.schedule import build_cdp_timeline, build_dp_timeline


def _as_executed(tl, unit=1000):
    # time step g occupies [g * unit, g * unit + unit - 1]
    return {(t.kind, t.micro_batch, t.stage, t.training_step): (t.start * unit, t.end * unit + unit - 1)
            for t in tl.tasks}


@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("scheme", ["dp", "cdp-v1", "cdp-v2"])
def test_plan_as_execution_reproduces_plan_accounting(n, scheme):
    steps = 4
    if scheme == "dp":
        tl = build_dp_timeline(ParallelismConfig(Scheme.MULTI_GPU_DP, n, 1, steps))
    else:
        tl = build_cdp_timeline(ParallelismConfig(Scheme.MULTI_GPU_CDP, n, 1, steps), rule_by_name(scheme, n))
    ex = _as_executed(tl)
    rb = [100 * j for j in range(1, n + 1)]
    act = executed_activation(ex, rb, steps)
    assert act.peak_bytes == _planned_peak(tl, rb)
    assert act.steady_min_bytes <= act.mean_bytes <= act.steady_max_bytes
    bal = executed_balance(tl, ex)
    assert bal["chain_order_violations"] == []
    if scheme != "dp":
        ref = balance_report(schedule_cdp_ring_reduce(tl, make_homogeneous_profile(n, n, n, 1)))
        assert bal["max_sends"] == ref.max_sends
        assert bal["max_sends_or_receives_per_worker"] == 1


def test_series_releases_before_acquires():
    from paper_2403_08837_b200.schedule import TaskKind as K

    ex = {(K.FORWARD, 1, 1, 1): (0, 5), (K.BACKWARD, 1, 1, 1): (6, 10),
          (K.FORWARD, 2, 1, 1): (10, 12), (K.BACKWARD, 2, 1, 1): (13, 20)}
    ser = activation_series_ns(ex, [7])
    assert max(v for _, v in ser) == 7  # the record released at t=10 is not counted with the one acquired at 10
