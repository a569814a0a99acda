"""Multi-GPU CDP protocol (P2P gradient hop over peer memory, fused update on
the last rank, parameter pulls), emulated with N rank trainers sharing one GPU
in one process: every rank has its own stream, shared region and flags, and
the kernels synchronise only through the system-scope flags — the exact code
path of one-process-per-GPU runs, minus NVLink.

The N-rank run performs the same arithmetic in the same order as the
single-GPU N-worker trainer (S_i = S_{i-1} + g_i, update on worker N), so the
parameters must agree bit for bit.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_ranks(task, rule_name, steps, dtype, momentum):
    from paper_2403_08837_b200.device import DeviceMlpTrainer
    from paper_2403_08837_b200.rules import rule_by_name

    n = task.n
    rule = None if rule_name == "dp" else rule_by_name(rule_name, n)
    ranks = [DeviceMlpTrainer.for_rank(task.model.dims, task.micro_batch_size, n, r, task.model.loss_code, rule,
                                       dtype=dtype, momentum=momentum, inputs=task.inputs, targets=task.targets)
             for r in range(n)]
    regions = [t.region() for t in ranks]
    init = np.concatenate(task.init_params())
    for t in ranks:
        t.set_params(init, which=-1)
        t.connect(regions)
    b = task.micro_batch_size
    for step in range(1, steps + 1):
        perm = task.permutation(step)
        for r, t in enumerate(ranks):  # launch every rank's step; they synchronise on device flags
            t.step(perm[r * b:(r + 1) * b], 0.05)
    for t in ranks:
        t.sync()
        assert t.ring_error() == 0
    losses = np.mean([t.history(steps)[0] for t in ranks], axis=0)
    final = ranks[-1].get_params(0)
    for t in ranks:
        t.close()
    return losses, final


def _run_single(task, rule_name, steps, dtype, momentum):
    from paper_2403_08837_b200.device import DeviceMlpTrainer
    from paper_2403_08837_b200.rules import rule_by_name

    rule = None if rule_name == "dp" else rule_by_name(rule_name, task.n)
    tr = DeviceMlpTrainer(task.model.dims, task.micro_batch_size, task.n, task.model.loss_code, rule, dtype=dtype,
                          momentum=momentum, inputs=task.inputs, targets=task.targets)
    tr.set_params(np.concatenate(task.init_params()), which=-1)
    for step in range(1, steps + 1):
        tr.step(task.permutation(step), 0.05)
    losses = tr.history(steps)[0]
    final = tr.get_params(0)
    tr.close()
    return losses, final


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("rule", ["cdp-v1", "cdp-v2", "dp"])
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_ranks_match_single_gpu_bit_exact(cuda, n, rule, dtype):
    from paper_2403_08837_b200.training import make_mlp_task

    task = make_mlp_task(n=n, micro_batch_size=8, seed=4, width=64, in_dim=96, out_dim=10, loss_kind="xent")
    l_multi, p_multi = _run_ranks(task, rule, 6, dtype, 0.9)
    l_single, p_single = _run_single(task, rule, 6, dtype, 0.9)
    assert np.array_equal(p_multi, p_single)
    assert np.allclose(l_multi, l_single, rtol=1e-12, atol=0)


def test_ranks_match_reference(cuda):
    """4 ranks, CDP-v2, fp32: against the fp64 oracle (tolerance of the fp32 mode)."""
    from oracle import engine as OE
    from paper_2403_08837_b200.training import make_mlp_task

    kw = dict(n=4, micro_batch_size=8, seed=6, width=64, in_dim=96, out_dim=10, loss_kind="xent")
    losses, final = _run_ranks(make_mlp_task(**kw), "cdp-v2", 8, "fp32", 0.9)
    ref = OE.run_experiment(OE.make_mlp_task(**kw), rules=("cdp-v2",), steps=8, lr=0.05, momentum=0.9)["cdp-v2"]
    want = np.concatenate(ref.final_params)
    assert np.linalg.norm(final - want) / np.linalg.norm(want) <= 1e-5
    assert np.all(np.abs(losses - np.array(ref.losses)) <= 1e-5 * np.abs(np.array(ref.losses)))


@pytest.mark.parametrize("n", [2, 4])
def test_grouped_layers_ranks_vs_oracle(cuda, n):
    """8 layers grouped into n stages (stage = contiguous layers, versions per stage,
    hops and pulls per layer): n ranks vs the single-GPU trainer (bit-exact) and vs
    the fp64 oracle with the rule expanded to layers."""
    from oracle import engine as OE
    from paper_2403_08837_b200.device import DeviceMlpTrainer
    from paper_2403_08837_b200.executor import layer_stages
    from paper_2403_08837_b200.rules import min_delay_rule
    from paper_2403_08837_b200.training import make_mlp_task

    kw = dict(n=8, micro_batch_size=16, seed=9, width=48, in_dim=64, out_dim=10, loss_kind="xent")
    base = make_mlp_task(**kw)
    ls = layer_stages(8, n)
    rule = min_delay_rule(n)
    inputs, targets = base.inputs[: n * 16], base.targets[: n * 16]
    steps = 5
    perms = [np.random.default_rng([1, t]).permutation(n * 16) for t in range(1, steps + 1)]
    init = np.concatenate(base.init_params())
    # single GPU, n workers
    tr = DeviceMlpTrainer(base.model.dims, 16, n, 1, rule, dtype="fp32", momentum=0.9, inputs=inputs,
                          targets=targets, layer_stage=ls)
    tr.set_params(init, -1)
    for t in range(steps):
        tr.step(perms[t], 0.05)
    single = tr.get_params(0)
    tr.close()
    # n ranks
    ranks = [DeviceMlpTrainer.for_rank(base.model.dims, 16, n, r, 1, rule, dtype="fp32", momentum=0.9,
                                       inputs=inputs, targets=targets, layer_stage=ls) for r in range(n)]
    regions = [r_.region() for r_ in ranks]
    for r_ in ranks:
        r_.set_params(init, -1)
        r_.connect(regions)
    for t in range(steps):
        for r, r_ in enumerate(ranks):
            r_.step(perms[t][r * 16:(r + 1) * 16], 0.05)
    for r_ in ranks:
        r_.sync()
        assert r_.ring_error() == 0
    multi = ranks[-1].get_params(0)
    for r_ in ranks:
        r_.close()
    assert np.array_equal(single, multi)
    # oracle: layer-expanded rule table
    otask = OE.make_mlp_task(**kw)
    fresh = [[rule.reads_fresh(i, ls[l]) for l in range(8)] for i in range(1, n + 1)]
    cur = otask.init_params()
    prev = [p.copy() for p in cur]
    vel = [np.zeros_like(p) for p in cur]
    for t in range(1, steps + 1):
        p = perms[t - 1]
        batches = [(inputs[p[i * 16:(i + 1) * 16]], targets[p[i * 16:(i + 1) * 16]]) for i in range(n)]
        new, _ = OE.advance(otask, cur, prev, t, batches, 0.05, fresh, 0.9, vel)
        prev, cur = cur, new
    want = np.concatenate(cur)
    assert np.linalg.norm(multi - want) / np.linalg.norm(want) <= 1e-5


@pytest.mark.parametrize("n", [2, 4])
def test_dp_allreduce_baseline_matches_single_gpu_dp(cuda, n):
    """DP all-reduce baseline (ref comm.py:70-90): every rank computes its micro-batch
    gradient (hop role 4), the sum is reduced (here in rank order on one device, as the
    ring does), every replica applies the update -> bit-identical to single-GPU DP."""
    import torch
    from paper_2403_08837_b200.device import DeviceMlpTrainer
    from paper_2403_08837_b200.training import make_mlp_task

    task = make_mlp_task(n=n, micro_batch_size=8, seed=4, width=64, in_dim=96, out_dim=10, loss_kind="xent")
    ranks = [DeviceMlpTrainer.for_rank(task.model.dims, 8, n, r, 1, None, dtype="bf16", momentum=0.9,
                                       inputs=task.inputs, targets=task.targets, allreduce=True) for r in range(n)]
    regions = [t.region() for t in ranks]
    init = np.concatenate(task.init_params())
    for t in ranks:
        t.set_params(init, -1)
        t.connect(regions)
    views = [t.partial_tensor() for t in ranks]
    for step in range(1, 6):
        perm = task.permutation(step)
        for r, t in enumerate(ranks):
            t.step(perm[r * 8:(r + 1) * 8], 0.05)
        for t in ranks:
            t.sync()
        total = views[0].clone()
        for v in views[1:]:
            total += v
        torch.cuda.synchronize()
        for t, v in zip(ranks, views):
            v.copy_(total)
            torch.cuda.synchronize()
            t.apply_update()
    finals = [t.get_params(0) for t in ranks]
    for t in ranks:
        t.close()
    single = _run_single(task, "dp", 5, "bf16", 0.9)[1]
    for f in finals:
        assert np.array_equal(f, finals[0])
    assert np.array_equal(finals[0], single)
