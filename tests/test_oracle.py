"""The CPU oracle is pinned against the reference itself (golden vectors).

oracle/cdp_oracle.c restates the reference's Cython kernel loop for loop, so
the comparison is exact equality, not a tolerance.  The engine restatement
reproduces the reference's run_experiment losses, final parameters and
version traces exactly on the toy tasks, and the first config-1 steps.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import engine as OE
from oracle import kernels as OK

KER = np.load(os.path.join(GOLDEN, "kernels.npz"))
TOY = np.load(os.path.join(GOLDEN, "toy_runs.npz"))
C1 = np.load(os.path.join(GOLDEN, "config1.npz"))


def _mlp_case(k):
    g = lambda s: KER[f"mlp{k}_{s}"]
    kind = int(g("kind"))
    y = g("y") if kind == 0 else None
    lab = g("labels") if kind == 1 else None
    return tuple(int(d) for d in g("dims")), g("theta"), g("x"), y, lab, kind, float(g("loss")), g("grad")


@pytest.mark.parametrize("k", range(int(KER["n_mlp"])))
def test_oracle_mlp_kernel_bit_exact(k):
    dims, th, x, y, lab, kind, loss, grad = _mlp_case(k)
    l2, g2 = OK.mlp_value_grad(dims, th, x, y, lab, kind)
    assert l2 == loss
    assert np.array_equal(g2, grad)


def test_oracle_quad_kernel_bit_exact():
    l2, g2 = OK.quad_value_grad(KER["quad_a"], KER["quad_theta"], KER["quad_targets"])
    assert l2 == float(KER["quad_loss"])
    assert np.array_equal(g2, KER["quad_grad"])


def test_reference_kernel_build_matches_golden():
    """oracle/_ref holds the reference's own kernel compiled from its source."""
    mod = OK.load_reference_kernels()
    if mod is None:
        pytest.skip("oracle/_ref not built (no /root/reference and no prebuilt module)")
    dims, th, x, y, lab, kind, loss, grad = _mlp_case(1)
    l2, g2 = mod.mlp_value_grad(dims, th, x, y, lab, kind)
    assert l2 == loss and np.array_equal(g2, grad)


TOY_TASKS = {
    "mlp_mse": lambda: OE.make_mlp_task(n=4, micro_batch_size=4, seed=3, width=8, in_dim=6, out_dim=3, loss_kind="mse"),
    "mlp_xent": lambda: OE.make_mlp_task(n=4, micro_batch_size=4, seed=5, width=8, in_dim=6, out_dim=3, loss_kind="xent"),
    "mlp_xent_n3": lambda: OE.make_mlp_task(n=3, micro_batch_size=6, seed=7, width=10, in_dim=5, out_dim=4,
                                            loss_kind="xent"),
    "quad": lambda: OE.make_quadratic_task(n=4, micro_batch_size=2, seed=11),
}


@pytest.mark.parametrize("name", list(TOY_TASKS))
def test_oracle_task_data_bit_exact(name):
    task = TOY_TASKS[name]()
    assert np.array_equal(task.inputs, TOY[f"{name}_inputs"])
    assert np.array_equal(task.targets, TOY[f"{name}_targets"])
    assert np.array_equal(np.concatenate(task.init_params()), TOY[f"{name}_init"])
    perm3 = np.concatenate([b[0].ravel() for b in task.micro_batches(3)])
    assert np.array_equal(perm3, TOY[f"{name}_perm3"])


@pytest.mark.parametrize("name", list(TOY_TASKS))
@pytest.mark.parametrize("mom", [0.0, 0.9])
def test_oracle_engine_bit_exact(name, mom):
    task = TOY_TASKS[name]()
    res = OE.run_experiment(task, steps=20, lr=0.05, momentum=mom, record_trace=True)
    for rule, run in res.items():
        key = f"{name}_m{int(mom * 10)}_{rule}"
        assert np.array_equal(np.array(run.losses), TOY[key + "_losses"])
        assert np.array_equal(np.concatenate(run.final_params), TOY[key + "_final"])
        assert np.array_equal(np.array(run.trace, dtype=np.int64), TOY[key + "_trace"])
        assert (run.diverged_at or -1) == int(TOY[key + "_diverged"])


def test_oracle_config1_first_steps_bit_exact():
    task = OE.make_mlp_task(n=4, micro_batch_size=32, seed=0, width=256, in_dim=3072, out_dim=10, loss_kind="xent")
    assert float(task.inputs.sum()) == float(C1["inputs_sum"])
    assert np.array_equal(task.targets, C1["targets"])
    assert np.array_equal(np.concatenate(task.init_params())[C1["sample_idx"]], C1["init_sample"])
    res = OE.run_experiment(task, steps=2, lr=0.05, momentum=0.9)
    for rule, run in res.items():
        assert np.array_equal(np.array(run.losses), C1[f"m9_{rule}_losses"][:2])
