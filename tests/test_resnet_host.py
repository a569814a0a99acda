"""ResNet model spec / layout / torch-CPU oracle on CPU (no GPU)."""

import numpy as np
import torch

from oracle.resnet_torch import CifarResNet, ResNetOracle, grads_flat, init_flat, load_flat
from paper_2403_08837_b200.resnet import RESNET18, flat_to_tensors, layer_specs, stage_partition, torch_to_flat


def test_resnet18_parameter_count_matches_torchvision_cifar():
    specs = layer_specs(**RESNET18)
    assert sum(int(np.prod(s)) for _, s, _ in specs) == 11_173_962
    assert len(specs) == 41


def test_layout_roundtrip():
    w, d = (64, 128), (1, 1)
    specs = layer_specs(w, d)
    flat = init_flat(w, d, seed=3)
    m = CifarResNet(w, d).double()
    load_flat(m, flat, specs)
    assert np.array_equal(torch_to_flat(m), flat)


def test_stage_partition_contiguous_and_balanced():
    specs = layer_specs(**RESNET18)
    for n in (1, 2, 4, 8):
        st = stage_partition(specs, n)
        assert list(st) == sorted(st) and set(st) == set(range(1, n + 1))
        fl = np.array([f for _, _, f in specs], dtype=float)
        per = [fl[st == k].sum() for k in range(1, n + 1)]
        assert max(per) <= 2.2 * fl.sum() / n


def test_oracle_gradients_match_autograd_layout():
    w, d = (64,), (1,)
    specs = layer_specs(w, d, hw=8)
    flat = init_flat(w, d, seed=1)
    orc = ResNetOracle(w, d, specs)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(4, 8, 8, 3))
    y = rng.integers(0, 10, size=4)
    loss, grads = orc.loss_and_grads(flat_to_tensors(flat, specs), x, y)
    # finite difference on one conv weight and one bn gamma
    eps = 1e-6
    for t_idx, k in ((0, 5), (1, 2)):
        f2 = flat.copy()
        base = sum(int(np.prod(s)) for _, s, _ in specs[:t_idx])
        f2[base + k] += eps
        l2, _ = orc.loss_and_grads(flat_to_tensors(f2, specs), x, y)
        assert abs((l2 - loss) / eps - grads[t_idx][k]) < 1e-4 * max(1.0, abs(grads[t_idx][k]))
