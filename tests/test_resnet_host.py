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


def test_resnet50_parameter_count_matches_torchvision():
    from paper_2403_08837_b200.resnet import RESNET50

    specs = layer_specs(**RESNET50, classes=1000, hw=224)
    assert sum(int(np.prod(s)) for _, s, _ in specs) == 25_557_032
    assert len(specs) == 107


def test_resnet50_layout_matches_torchvision_order():
    """Our tensor order / shapes == torchvision.models.resnet50 named_parameters (conv/bn/fc)."""
    import torchvision

    from paper_2403_08837_b200.resnet import RESNET50

    tv = torchvision.models.resnet50(num_classes=1000)
    shapes = []
    for name, p in tv.named_parameters():
        if name.endswith("bn1.bias") or ".bn" in name and name.endswith("bias") or name.endswith("downsample.1.bias"):
            continue
        shapes.append(tuple(p.shape))
    ours = []
    for kind, shape, _ in layer_specs(**RESNET50, classes=1000, hw=224):
        if kind == "conv":
            r, s, cin, cout = shape
            ours.append((cout, cin, r, s))
        elif kind == "bn":
            ours.append((shape[0] // 2,))
        else:
            ours.append((shape[1], shape[0] - 1))
            ours.append((shape[1],))
    assert ours == shapes


def test_bottleneck_imagenet_layout_roundtrip():
    from oracle.resnet_torch import TorchResNet

    w, d = (64, 128), (1, 1)
    specs = layer_specs(w, d, hw=32, block="bottleneck", stem="imagenet")
    flat = init_flat(w, d, seed=3, block="bottleneck", stem="imagenet")
    assert flat.size == sum(int(np.prod(s)) for _, s, _ in specs)
    m = TorchResNet(w, d, 10, "bottleneck", "imagenet").double()
    load_flat(m, flat, specs)
    assert np.array_equal(torch_to_flat(m), flat)


def test_pull_chain_follows_the_reader_order():
    """Theta forwarding: per stage, the readers (ranks 0..N-2) form one chain - fresh readers in worker order,
    then stale ones - whose head pulls from the updater; each reader serves exactly its successor."""
    from paper_2403_08837_b200.resnet import pull_chain
    from paper_2403_08837_b200.rules import rule_by_name

    for n in (2, 3, 4, 8):
        for rule in (None, rule_by_name("cdp-v1", n), rule_by_name("cdp-v2", n)):
            ch = [pull_chain(rule, n, r) for r in range(n - 1)]
            for j in range(n):
                heads = [r for r in range(n - 1) if ch[r][j, 0] == -1]
                assert len(heads) == 1
                order, r = [], heads[0]
                while r != -1:
                    order.append(r)
                    nxt = int(ch[r][j, 1])
                    if nxt != -1:
                        assert ch[nxt][j, 0] == r
                    r = nxt
                assert sorted(order) == list(range(n - 1))
                fresh = [rule is None or rule.reads_fresh(r + 1, j + 1) for r in order]
                assert fresh == sorted(fresh, reverse=True)  # fresh readers first
