"""Plan layer vs the reference, bit-exact.

Every timeline, comm event, validator verdict, gradient-reduction replay,
balance report and measured activation peak recorded from the reference by
tests/golden/make_golden.py must be reproduced exactly by
paper_2403_08837_b200's own plan code.
"""

import gzip
import json
import os
from fractions import Fraction

import pytest

from conftest import GOLDEN
from paper_2403_08837_b200 import (
    CostWeights,
    ModelProfile,
    ParallelismConfig,
    Scheme,
    build_cdp_timeline,
    build_dp_timeline,
    build_zero_timeline,
    generic_rule,
    make_homogeneous_profile,
    validate_timeline,
)
from paper_2403_08837_b200.comm import balance_report, scheduled_timeline, verify_gradient_reduction
from paper_2403_08837_b200.costs import peak_activation

with gzip.open(os.path.join(GOLDEN, "plans.json.gz"), "rt") as fh:
    CASES = json.load(fh)

GENERIC = [[False, False, True], [False, True, True], [False, False, False]]


def _enc_task(t):
    return [t.kind.value, t.micro_batch, t.stage, t.training_step, t.param_version, t.device, t.start, t.duration]


def _enc_event(e):
    return [e.boundary, e.kind.value, e.src, e.dst, str(e.payload), e.stage, e.micro_batch, e.participants, e.depth]


def _build(name):
    """Rebuild the case `name` with our code (same naming as make_golden.py)."""
    if name.startswith("generic") or name.startswith("sched-generic"):
        cfg = ParallelismConfig(Scheme.MULTI_GPU_CDP, 3, 2, 3)
        prof = ModelProfile((5, 7, 11), (30, 20, 10), 12)
        rule = generic_rule(GENERIC)
        tl = scheduled_timeline(cfg, prof, rule) if name.startswith("sched") else build_cdp_timeline(cfg, rule)
        return tl, prof
    parts = name.split("-")
    sched = parts[0] == "sched"
    zero = parts[0] == "zero"
    if sched or zero:
        parts = parts[1:]
    # scheme value is the leading tokens up to the rule / n
    tokens = "-".join(parts)
    scheme = next(s for s in sorted(Scheme, key=lambda s: -len(s.value)) if tokens.startswith(s.value + "-"))
    rest = tokens[len(scheme.value) + 1:].split("-")
    rule = None
    if rest[0] == "cdp":
        rule = "-".join(rest[:2])
        rest = rest[2:]
    n = int(rest[0][1:])
    steps = int(rest[1][1:])
    w = (int(rest[2][1]), int(rest[2][2])) if len(rest) > 2 else (1, 1)
    cfg = ParallelismConfig(scheme, n, 2, steps, CostWeights(*w))
    prof = make_homogeneous_profile(n, 12 * n, 60 * n, 0)
    if sched:
        return (scheduled_timeline(cfg, prof, rule) if rule else scheduled_timeline(cfg, prof)), prof
    if zero:
        return build_zero_timeline(cfg, prof, scheme is Scheme.ZERO_CDP), prof
    if rule:
        return build_cdp_timeline(cfg, rule), prof
    return build_dp_timeline(cfg), prof


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_plan_matches_reference(case):
    if "error" in case:
        with pytest.raises(Exception) as err:
            _build(case["name"])
        assert type(err.value).__name__ == case["error"]
        return
    tl, prof = _build(case["name"])
    assert tl.horizon == case["horizon"]
    assert [[d.id, d.gpu, d.capacity, d.param_model.value, list(d.owned_stages)] for d in tl.devices] == case["devices"]
    assert [_enc_task(t) for t in tl.tasks] == case["tasks"]
    assert [_enc_event(e) for e in tl.comm_events] == case["events"]
    assert [[v.kind, v.message] for v in validate_timeline(tl).violations] == case["violations"]
    assert list(tl.steady_window()) == case["steady"]
    if "reduction" in case:
        got = [[c.stage, c.training_step, c.complete_at, c.first_fresh_read, c.ok] for c in verify_gradient_reduction(tl)]
        assert got == case["reduction"]
        br = balance_report(tl)
        assert [br.max_sends, br.min_sends, str(br.mean_sends), list(br.deep_boundaries),
                list(br.cyclic_depth_flags)] == case["balance"]
    if "peak_activation" in case:
        assert peak_activation(tl, prof) == Fraction(case["peak_activation"])
