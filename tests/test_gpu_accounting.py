"""Accounting on executed schedules (ref costs.py:191-329 measure_costs,
comm.py:196-221 balance_report): the activation and hop fields computed from the device's own
%globaltimer stamps of a single-GPU cyclic run (4 worker streams, MLP executor), against the plan."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(rule_name, steps=4, n=4, batch=16, width=64):
    from paper_2403_08837_b200.accounting import executed_activation, executed_balance
    from paper_2403_08837_b200.cli import _planned_peak
    from paper_2403_08837_b200.device import DeviceMlpTrainer
    from paper_2403_08837_b200.profiles import ParallelismConfig, Scheme
    from paper_2403_08837_b200.rules import rule_by_name
    from paper_2403_08837_b200.schedule import build_cdp_timeline, build_dp_timeline
    from paper_2403_08837_b200.training import make_mlp_task

    task = make_mlp_task(n=n, micro_batch_size=batch, seed=0, width=width, in_dim=width, out_dim=10,
                         loss_kind="xent")
    rule = None if rule_name == "dp" else rule_by_name(rule_name, n)
    tr = DeviceMlpTrainer(task.model.dims, batch, n, 1, rule, dtype="bf16", inputs=task.inputs,
                          targets=task.targets)
    tr.set_params(np.concatenate(task.init_params()), which=-1)
    executed = {}
    for t in range(1, steps + 1):
        executed.update(tr.trace_step(task.permutation(t), 0.05, t))
    tr.close()
    cfg = ParallelismConfig(Scheme.SINGLE_GPU_DP if rule is None else Scheme.SINGLE_GPU_CDP, n, batch, steps)
    tl = build_dp_timeline(cfg) if rule is None else build_cdp_timeline(cfg, rule)
    rb = [batch * ((d + 15) // 16 * 16) * 2 for d in task.model.dims[:-1]]
    return executed_activation(executed, rb, steps), _planned_peak(tl, rb), executed_balance(tl, executed), rb


def test_executed_activation_and_hops_cdp_vs_dp(cuda):
    res = {r: _run(r) for r in ("dp", "cdp-v2", "cdp-v1")}
    for name, (act, planned, bal, rb) in res.items():
        # the executor's record slots are the plan's interval colouring: the device can never hold more
        # live records than the plan's peak
        assert 0 < act.peak_bytes <= planned, (name, act, planned)
        assert act.steady_min_bytes <= act.mean_bytes <= act.steady_max_bytes <= act.peak_bytes
        # every worker sends and receives at most one gradient hop per boundary; hops follow the chain
        assert bal["max_sends_or_receives_per_worker"] == 1, (name, bal)
        assert bal["chain_order_violations"] == [], bal["chain_order_violations"][:3]
    # single-GPU CDP holds fewer records than DP at peak (ref costs.py:111-115: (N+1)/2 vs N)
    assert res["cdp-v2"][0].peak_bytes < res["dp"][0].peak_bytes
    assert res["cdp-v1"][0].peak_bytes < res["dp"][0].peak_bytes
    # DP hops all workers at one boundary, CDP spreads them (max sends per boundary N vs <= N/2 + 1)
    assert res["dp"][2]["max_sends"] == 4 and res["cdp-v2"][2]["max_sends"] <= 3


def test_cli_trace_writes_accounting(cuda, tmp_path):
    from paper_2403_08837_b200.cli import main

    rc = main(["trace", "--n", "4", "--batch", "16", "--width", "64", "--training-steps", "4", "--rule", "cdp-v2",
               "--out", str(tmp_path)])
    assert rc == 0
    rep = json.loads((tmp_path / "accounting.json").read_text())
    assert rep["executed"]["peak_activation_bytes"] <= rep["planned_peak_activation_bytes"]
    assert rep["balance"]["chain_order_violations"] == []
