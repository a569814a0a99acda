"""Memory / state-volume closed forms of the hot-path schemes (costs.closed_form_memory) against the
reference's own closed_form_costs (ref costs.py:64-153; golden tests/golden/closed_form.json made by
tests/golden/make_golden.py from the unmodified reference): single-GPU DP N*B*Psi_A vs CDP (N+1)/2*B*Psi_A,
multi-GPU B*Psi_A, ZeRO-DP 2*Psi_P vs ZeRO-CDP 2(N-1)/N*Psi_P per device per step."""

import json
import os
from fractions import Fraction

from paper_2403_08837_b200.costs import closed_form_memory
from paper_2403_08837_b200.profiles import ParallelismConfig, Scheme, make_homogeneous_profile

GOLD = os.path.join(os.path.dirname(__file__), "golden", "closed_form.json")


def test_closed_form_memory_matches_reference():
    rows = json.load(open(GOLD))
    assert len(rows) == 270
    for scheme, n, b, pp, pa, act, state in rows:
        prof = make_homogeneous_profile(n, pp, pa, 1)
        r = closed_form_memory(ParallelismConfig(Scheme(scheme), n, b, 3), prof)
        assert r.activation_per_device == Fraction(act), (scheme, n, b, pp, pa)
        assert r.state_volume_per_device == Fraction(state), (scheme, n, b, pp, pa)


def test_cdp_single_gpu_ratio():
    prof = make_homogeneous_profile(4, 48, 240, 1)
    dp = closed_form_memory(ParallelismConfig(Scheme.SINGLE_GPU_DP, 4, 2, 3), prof).activation_per_device
    cdp = closed_form_memory(ParallelismConfig(Scheme.SINGLE_GPU_CDP, 4, 2, 3), prof).activation_per_device
    assert cdp / dp == Fraction(5, 8)  # (N+1)/(2N) at N = 4 (the 0.625 the ViT bench line is compared with)
