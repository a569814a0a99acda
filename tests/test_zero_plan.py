"""ZeRO-CDP device protocol (paper_2403_08837_b200/zero.py) vs the reference-parity state-transfer plan
(ref comm.py:93-144 over schedule.py:433-472).

Every use of a stage must obtain the same state as in the reference plan: its predecessor (the holder it
copies from) is the reference's previous user of the stage; the device reads the locally held initial
state only where the reference's holder still holds the initial state (no update of that stage yet).
After the first update the device's copies are exactly the reference's STATE_TRANSFER events."""

import pytest

from paper_2403_08837_b200.profiles import ParallelismConfig, Scheme, make_homogeneous_profile
from paper_2403_08837_b200.schedule import TaskKind, build_zero_timeline
from paper_2403_08837_b200.zero import KINDS, reference_transfers, state_bytes_per_step, transfers, zero_plan


def _timeline(n, steps):
    cfg = ParallelismConfig(scheme=Scheme.ZERO_CDP, n=n, training_steps=steps)
    return build_zero_timeline(cfg, make_homogeneous_profile(n, n, n, 1), cyclic=True)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
def test_every_use_reads_the_reference_state(n):
    steps = 5
    plan = zero_plan(n)
    tl = _timeline(n, steps)
    for s in range(1, n + 1):
        uses = sorted((t for t in tl.tasks if t.stage == s), key=lambda t: t.start)
        first_update = next(t.start for t in uses if t.kind is TaskKind.BACKWARD and t.micro_batch == n)
        by_key = {(t.kind, t.micro_batch, t.training_step): t for t in uses}
        for k, t in enumerate(uses):
            if t.training_step == steps:
                continue  # the reference's final step has no step-(T+1) forwards (the device drains them)
            ki = KINDS.index(t.kind)
            i = t.micro_batch - 1
            ref_pred = uses[k - 1] if k > 0 else None
            pt = t.training_step + int(plan.dstep[s - 1, ki, i])
            if pt >= 1:
                pk = KINDS.index(ref_pred.kind) if ref_pred else None
                assert ref_pred is not None
                assert int(plan.prev[s - 1, ki, i]) == ref_pred.micro_batch - 1
                assert pt == ref_pred.training_step
                # the use index arithmetic points at that very task
                u = int(plan.base[s - 1, ki, i]) + (t.training_step - 1) * plan.uses_per_step
                pu = int(plan.base[s - 1, pk, ref_pred.micro_batch - 1]) + (pt - 1) * plan.uses_per_step
                assert pu == u - 1
            else:
                assert ref_pred is None or ref_pred.start < first_update
            assert by_key[(t.kind, t.micro_batch, t.training_step)] is t


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_copies_after_first_update_equal_reference_transfers(n):
    steps = 5
    plan = zero_plan(n)
    ours = set(e for e in transfers(plan, steps) if 3 <= e[0] < steps)
    ref = set(e for e in reference_transfers(n, steps) if 3 <= e[0] < steps)
    assert ours == ref and ours


@pytest.mark.parametrize("n", [2, 4, 8])
def test_received_units_per_step(n):
    """Each rank receives every stage at most twice per step (F and B uses); middle stages twice,
    summed over ranks the steady-state number of copies per step equals the reference event count."""
    plan = zero_plan(n)
    per_rank = [state_bytes_per_step(plan, [1] * n, r, momentum=False) // 8 for r in range(n)]
    assert all(u <= 2 * n for u in per_rank)
    ref_step = [e for e in reference_transfers(n, 5) if e[0] == 4]
    assert sum(per_rank) == len(ref_step)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_drain_units_are_next_step_forward_predecessors(n):
    from paper_2403_08837_b200.zero import drain_units

    plan = zero_plan(n)
    got = {(s, r) for r in range(n) for s in drain_units(plan, r)}
    want = {(s + 1, int(plan.prev[s, 1, j])) for s in range(n) for j in range(n) if int(plan.dstep[s, 1, j]) == 1}
    assert got == want


def test_frame_drain_plan():
    """End-of-run drain of the ZeRO-CDP state frames: the next-step forward copies the last frame reuses wait
    for (N = 4: w1's F3 / F4, w2's F3), derivable for N = 2..8 (every needed copy's predecessors are
    earlier steps or drained forwards — the planner raises otherwise)."""
    from paper_2403_08837_b200.zero import frame_drain_plan

    assert frame_drain_plan(2) == [[], []]
    assert frame_drain_plan(3) == [[(3, 0, 0, 0, -1)], [], []]
    assert frame_drain_plan(4) == [[(3, 0, 0, 0, -1), (4, 1, 1, -1, 0)], [(3, 0, 0, 0, -1)], [], []]
    for n in (5, 6, 8):
        plan = frame_drain_plan(n)
        assert len(plan) == n and not plan[-1] and not plan[-2]  # the last ranks drain nothing
        for rows in plan:
            assert [r[0] for r in rows] == sorted(r[0] for r in rows)  # use order


def test_zero_partition_is_block_aligned():
    from paper_2403_08837_b200.resnet import RESNET50, block_starts, layer_specs, zero_partition

    W, D = RESNET50["widths"], RESNET50["depths"]
    starts = set(block_starts(W, D, "bottleneck", "imagenet"))
    specs = layer_specs(W, D, 3, 224, "bottleneck", "imagenet", 1000)
    for n in (2, 4, 8):
        st = zero_partition(W, D, 224, "bottleneck", "imagenet", 1000, n)
        assert len(st) == len(specs) and st[0] == 1 and st[-1] == n
        cuts = [i for i in range(1, len(st)) if st[i] != st[i - 1]]
        assert len(cuts) == n - 1 and set(cuts) <= starts
