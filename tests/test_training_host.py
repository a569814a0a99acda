"""Host side of the training API on CPU: task data, initial parameters and
micro-batch partitions are bit-identical to the reference's (golden vectors),
rule resolution / errors follow engine.py:51-63, and no GPU is touched."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2403_08837_b200.rules import max_delay_rule, min_delay_rule
from paper_2403_08837_b200.training import make_mlp_task, make_quadratic_task
from paper_2403_08837_b200.training.engine import _resolve_rule, raise_for_flags
from paper_2403_08837_b200.training.models import NonFiniteGradientError

TOY = np.load(os.path.join(GOLDEN, "toy_runs.npz"))
C1 = np.load(os.path.join(GOLDEN, "config1.npz"))

TASKS = {
    "mlp_mse": lambda: make_mlp_task(n=4, micro_batch_size=4, seed=3, width=8, in_dim=6, out_dim=3, loss_kind="mse"),
    "mlp_xent": lambda: make_mlp_task(n=4, micro_batch_size=4, seed=5, width=8, in_dim=6, out_dim=3, loss_kind="xent"),
    "mlp_xent_n3": lambda: make_mlp_task(n=3, micro_batch_size=6, seed=7, width=10, in_dim=5, out_dim=4,
                                         loss_kind="xent"),
    "quad": lambda: make_quadratic_task(n=4, micro_batch_size=2, seed=11),
}


@pytest.mark.parametrize("name", list(TASKS))
def test_task_data_bit_identical_to_reference(name):
    task = TASKS[name]()
    assert np.array_equal(task.inputs, TOY[f"{name}_inputs"])
    assert np.array_equal(task.targets, TOY[f"{name}_targets"])
    assert np.array_equal(np.concatenate(task.init_params()), TOY[f"{name}_init"])
    assert np.array_equal(np.concatenate([b[0].ravel() for b in task.micro_batches(3)]), TOY[f"{name}_perm3"])


def test_config1_data_bit_identical():
    task = make_mlp_task(n=4, micro_batch_size=32, seed=0, width=256, in_dim=3072, out_dim=10, loss_kind="xent")
    assert float(task.inputs.sum()) == float(C1["inputs_sum"])
    assert np.array_equal(task.inputs.ravel()[::997], C1["inputs_sample"])
    assert np.array_equal(task.targets, C1["targets"])
    assert np.array_equal(np.concatenate(task.init_params())[C1["sample_idx"]], C1["init_sample"])
    first = np.concatenate([task.micro_batches(t)[0][0][:, 0] for t in (1, 2, 7)])
    assert np.array_equal(first, C1["perm_step"])


def test_rule_resolution_like_reference():
    assert _resolve_rule("dp", 4) is None
    assert _resolve_rule("v1", 4) == max_delay_rule(4)
    assert _resolve_rule("cdp-v2", 4) == min_delay_rule(4)
    with pytest.raises(ValueError):
        _resolve_rule("cdp-v3", 4)
    with pytest.raises(ValueError):
        _resolve_rule(min_delay_rule(3), 4)


def test_flag_mapping():
    raise_for_flags((0, 0, 0))
    with pytest.raises(NonFiniteGradientError) as e:
        raise_for_flags((0b0110, 1, 0))
    assert e.value.stage == 2
    with pytest.raises(NonFiniteGradientError) as e:
        raise_for_flags((0, 1, 0))
    assert e.value.stage == 0
    with pytest.raises(NonFiniteGradientError) as e:
        raise_for_flags((0, 0, 0b1000))
    assert e.value.stage == 4 and "update" in str(e.value)
