"""Single-GPU cyclic CDP for the ViT (BASELINE configs[3]; north star (1): N micro-batches on one GPU).

The trainer steps the reference's SINGLE_GPU_CDP / SINGLE_GPU_DP timeline (ref schedule.py:178-257,
every worker on gpu 0) with activation records from the plan's interval colouring
(executor.compile_segment_plan).  Checked here:

* parity with the float64 torch-CPU restatement under the reference's `_advance` (oracle/vit_torch.py)
  for DP, CDP-v1 and CDP-v2 at 2-4 workers (bf16 tolerances of tests/test_gpu_vit.py);
* bit-identity with the one-worker-per-rank ring on the same GPU (same stages): the cyclic executor
  changes when work runs and where records live, not the arithmetic;
* the memory claim of ref costs.py:111-115: the device's live-record high-water mark equals the plan's
  time-resolved peak, CDP's is ~(N+1)/(2N) of DP's;
* the executed versions (trace mode) against the rule table and the plan's schedule_consistency_check.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = dict(image=32, patch=8, dim=128, depth=2, heads=2, mlp=256, classes=10)
MB = 4


def _data(n, cfg, steps):
    from oracle.vit_torch import init_flat
    from paper_2403_08837_b200.resnet import synthetic_cifar

    x, y = synthetic_cifar(n * MB * 2, seed=4, hw=cfg["image"], classes=cfg["classes"])
    init = init_flat(**cfg, seed=0)
    perms = [np.random.default_rng([6, t]).permutation(len(x))[: n * MB] for t in range(1, steps + 1)]
    return x, y, init, perms


def _cyclic(n, rule, steps, cfg=CFG, trace=False, lr=0.1, dtype="bf16"):
    from paper_2403_08837_b200.vit import DeviceVit

    x, y, init, perms = _data(n, cfg, steps)
    tr = DeviceVit.single_gpu(cfg, MB, n, rule, 0.9, inputs=x, labels=y, trace=trace, dtype=dtype)
    tr.set_params(init, -1)
    for k in range(steps):
        tr.step(perms[k], lr)
    tr.sync()
    losses, flags = tr.history(steps)
    assert not flags.any()
    out = dict(x=x, y=y, init=init, perms=perms, losses=losses, final=tr.get_params(0).astype(np.float64),
               stage=tr.stage, stats=tr.stats(), plan=tr.plan, units=tr.units)
    if trace:
        out["recs"] = tr.access_trace()
    tr.close()
    return out


@pytest.mark.parametrize("n,rule_name", [(2, None), (2, "cdp-v1"), (2, "cdp-v2"), (3, "cdp-v2"), (4, "cdp-v1"),
                                         (4, "cdp-v2"), (4, None)])
def test_cyclic_vit_vs_restatement(cuda, n, rule_name):
    from oracle.vit_torch import run_cdp
    from paper_2403_08837_b200.rules import rule_by_name

    rule = rule_by_name(rule_name, n) if rule_name else None
    _vs_restatement(n, rule, "bf16", 2.5e-2, 5e-3)


def _vs_restatement(n, rule, dtype, tol_upd, tol_loss):
    from oracle.vit_torch import run_cdp

    r = _cyclic(n, rule, 3, dtype=dtype)
    fresh = None if rule is None else [[rule.reads_fresh(i, int(s)) for s in r["stage"]] for i in range(1, n + 1)]
    want, wl = run_cdp(CFG, r["init"], r["x"].astype(np.float64), r["y"], n, MB, r["perms"], 0.1, 0.9, fresh)
    d_ours, d_want = r["final"] - r["init"], want - r["init"]
    rel = float(np.linalg.norm(d_ours - d_want) / np.linalg.norm(d_want))
    print(f"update rel-L2 {rel:.2e}, max loss rel "
          f"{float(np.max(np.abs(r['losses'] - np.array(wl)) / np.abs(np.array(wl)))):.2e}")
    assert rel <= tol_upd, rel
    assert np.all(np.abs(r["losses"] - np.array(wl)) <= tol_loss * np.abs(np.array(wl))), (r["losses"], wl)


@pytest.mark.parametrize("n,rule_name", [(2, "cdp-v1"), (3, "cdp-v2"), (4, "cdp-v2"), (4, None)])
def test_cyclic_vit_fp32_vs_restatement(cuda, n, rule_name):
    """fp32 mode (3xTF32 operands, fp32 softmax) at the north star's fp32 tolerance: update rel-L2 <= 1e-5,
    losses within 5e-6 relative (measured 1.2e-6 - 2.4e-6 and <= 4e-7)."""
    from paper_2403_08837_b200.rules import rule_by_name

    rule = rule_by_name(rule_name, n) if rule_name else None
    _vs_restatement(n, rule, "fp32", 1e-5, 5e-6)


@pytest.mark.parametrize("n,rule_name", [(2, "cdp-v2"), (3, "cdp-v1"), (4, "cdp-v2")])
def test_cyclic_vit_equals_rank_ring(cuda, n, rule_name):
    """The single-GPU executor and the one-worker-per-rank ring (N trainers on this GPU, peer-memory
    hops) compute bit-identical parameters and losses."""
    from paper_2403_08837_b200.rules import rule_by_name
    from paper_2403_08837_b200.vit import DeviceVit

    rule = rule_by_name(rule_name, n)
    steps = 3
    r = _cyclic(n, rule, steps)
    tr = [DeviceVit(CFG, MB, n, k, rule, 0.9, inputs=r["x"], labels=r["y"], stage_of_unit=r["stage"])
          for k in range(n)]
    regions = [t.region() for t in tr]
    for t in tr:
        t.set_params(r["init"], -1)
        t.connect(regions)
    for k in range(steps):
        for i, t in enumerate(tr):
            t.step(r["perms"][k][i * MB:(i + 1) * MB], 0.1)
    for t in tr:
        t.sync()
        assert t.ring_error() == 0
    ring_final = tr[-1].get_params(0).astype(np.float64)
    ring_losses = np.array([t.history(steps)[0] for t in tr])
    for t in tr:
        t.close()
    assert np.array_equal(ring_final, r["final"])
    want = np.zeros(steps)
    for i in range(n):  # mean_i loss_i in ascending i (ref engine.py:113-116)
        want += ring_losses[i]
    assert np.allclose(r["losses"], want / n, rtol=1e-12, atol=0)


def test_cyclic_vit_activation_peak(cuda):
    """Executed high-water mark of live activation records (device counter around every record
    acquire / release) = the plan's time-resolved peak; CDP holds ~(N+1)/(2N) of DP's records
    (ref costs.py:111-115: (N+1)/2 vs N micro-batches)."""
    from paper_2403_08837_b200.rules import rule_by_name

    cfg = dict(CFG, depth=6)
    n = 4
    res = {}
    for name in ("dp", "cdp-v2"):
        rule = None if name == "dp" else rule_by_name(name, n)
        r = _cyclic(n, rule, 2, cfg=cfg)
        st, plan = r["stats"], r["plan"]
        rb = st["record_bytes"]
        assert st["record_slots"] == [int(v) for v in plan.pools]
        assert st["activation_bytes"] == sum(int(p) * b for p, b in zip(plan.pools, rb))
        assert st["live_record_high_water_bytes"] == plan.peak_bytes(rb)
        res[name] = st["live_record_high_water_bytes"]
        if name == "dp":  # lockstep DP keeps every worker's whole record set alive at the turn
            assert st["record_slots"] == [n, n * cfg["depth"], n]
    ratio = res["cdp-v2"] / res["dp"]
    assert ratio <= (n + 1) / (2 * n) + 0.02, ratio


@pytest.mark.parametrize("n,rule_name", [(3, "cdp-v2"), (4, "cdp-v1"), (3, None)])
def test_cyclic_vit_executed_versions(cuda, n, rule_name):
    from paper_2403_08837_b200 import ParallelismConfig, Scheme, build_cdp_timeline, build_dp_timeline
    from paper_2403_08837_b200.rules import rule_by_name
    from paper_2403_08837_b200.training import schedule_consistency_check

    rule = rule_by_name(rule_name, n) if rule_name else None
    steps = 3
    r = _cyclic(n, rule, steps, trace=True)
    recs, stage = r["recs"], r["stage"]
    n_units = len(r["units"])
    seen = set()
    for rec in recs:
        t, w, unit, kind, phase, slot, v = (int(rec[k]) for k in rec.dtype.names)
        i, j = w + 1, int(stage[unit - 1])
        want = (t if rule is None else rule.version_read(i, j, t)) if kind in (0, 1) else (t if kind == 2 else t + 1)
        if kind >= 2:
            assert i == n, "only the last worker updates"
        assert v == want and slot == (want & 1), dict(t=t, worker=i, unit=unit, kind=kind, v=v, want=want)
        seen.add((t, i, unit, kind))
    for t in range(1, steps + 1):
        for i in range(1, n + 1):
            for u in range(1, n_units + 1):
                assert (t, i, u, 0) in seen
        for u in range(1, n_units + 1):
            assert (t, n, u, 2) in seen and (t, n, u, 3) in seen
    trace = sorted({(int(q["t"]), int(q["rank"]) + 1, int(stage[int(q["unit"]) - 1]), int(q["version"]))
                    for q in recs if q["kind"] == 0})
    cfg = ParallelismConfig(Scheme.SINGLE_GPU_DP if rule is None else Scheme.SINGLE_GPU_CDP, n, 1, steps)
    tl = build_dp_timeline(cfg) if rule is None else build_cdp_timeline(cfg, rule)
    ok, bad = schedule_consistency_check(tl, trace)
    assert ok, bad
    assert {(t.training_step, t.micro_batch, t.stage) for t in tl.tasks if t.kind.name == "FORWARD"} == \
        {(t, i, j) for t, i, j, _ in trace}
