"""ViT restatement (oracle/vit_torch.py) pinned to torchvision's VisionTransformer (the model BASELINE
configs[3] names) on the same parameters; parameter count of ViT-B/16."""

import numpy as np
import torch

from oracle.vit_torch import VitOracle, init_flat, vit_loss, vit_specs

CFG = dict(image=32, patch=8, dim=64, depth=2, heads=2, mlp=128, classes=10)


def test_vit_b16_parameter_count():
    specs = vit_specs()
    assert sum(int(np.prod(s)) for _, s in specs) == 86_567_656
    assert len(specs) == 3 + 6 * 12 + 2


def _to_torchvision(flat, cfg):
    import torchvision

    m = torchvision.models.VisionTransformer(image_size=cfg["image"], patch_size=cfg["patch"], num_layers=cfg["depth"],
                                             num_heads=cfg["heads"], hidden_dim=cfg["dim"], mlp_dim=cfg["mlp"],
                                             num_classes=cfg["classes"]).double()
    specs = vit_specs(**cfg)
    parts, pos = {}, 0
    for name, shape in specs:
        n = int(np.prod(shape))
        parts[name] = torch.from_numpy(flat[pos:pos + n].reshape(shape).copy())
        pos += n
    P, D = cfg["patch"], cfg["dim"]
    with torch.no_grad():
        w = parts["patch"][:-1].reshape(P, P, 3, D).permute(3, 2, 0, 1)
        m.conv_proj.weight.copy_(w)
        m.conv_proj.bias.copy_(parts["patch"][-1])
        m.class_token.copy_(parts["cls"].reshape(1, 1, D))
        m.encoder.pos_embedding.copy_(parts["pos"].unsqueeze(0))
        for i, blk in enumerate(m.encoder.layers):
            for ln, key in ((blk.ln_1, "ln1"), (blk.ln_2, "ln2")):
                g = parts[f"b{i}.{key}"]
                ln.weight.copy_(g[:D])
                ln.bias.copy_(g[D:])
            qkv = parts[f"b{i}.qkv"]
            blk.self_attention.in_proj_weight.copy_(qkv[:-1].T)
            blk.self_attention.in_proj_bias.copy_(qkv[-1])
            pr = parts[f"b{i}.proj"]
            blk.self_attention.out_proj.weight.copy_(pr[:-1].T)
            blk.self_attention.out_proj.bias.copy_(pr[-1])
            f1, f2 = parts[f"b{i}.fc1"], parts[f"b{i}.fc2"]
            blk.mlp[0].weight.copy_(f1[:-1].T)
            blk.mlp[0].bias.copy_(f1[-1])
            blk.mlp[3].weight.copy_(f2[:-1].T)
            blk.mlp[3].bias.copy_(f2[-1])
        g = parts["ln"]
        m.encoder.ln.weight.copy_(g[:D])
        m.encoder.ln.bias.copy_(g[D:])
        h = parts["head"]
        m.heads.head.weight.copy_(h[:-1].T)
        m.heads.head.bias.copy_(h[-1])
    return m.eval()


def test_restatement_equals_torchvision_vit():
    flat = init_flat(**CFG, seed=1)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(3, 32, 32, 3))
    y = rng.integers(0, 10, size=3)
    ours = vit_loss(torch.from_numpy(flat), torch.from_numpy(x), torch.from_numpy(y), **CFG)
    tv = _to_torchvision(flat, CFG)
    ref = torch.nn.functional.cross_entropy(tv(torch.from_numpy(x).permute(0, 3, 1, 2).contiguous()),
                                            torch.from_numpy(y))
    assert abs(float(ours) - float(ref)) < 1e-10


def test_oracle_gradients_finite_difference():
    flat = init_flat(**CFG, seed=2)
    orc = VitOracle(CFG)
    rng = np.random.default_rng(1)
    x = rng.normal(size=(2, 32, 32, 3))
    y = rng.integers(0, 10, size=2)
    sizes = orc.sizes
    parts = np.split(flat, np.cumsum(sizes)[:-1])
    loss, grads = orc.loss_and_grads(parts, x, y)
    eps = 1e-6
    for t_idx, k in ((0, 7), (4, 11), (len(sizes) - 1, 3)):
        f2 = flat.copy()
        base = int(np.sum(sizes[:t_idx]))
        f2[base + k] += eps
        l2, _ = orc.loss_and_grads(np.split(f2, np.cumsum(sizes)[:-1]), x, y)
        assert abs((l2 - loss) / eps - grads[t_idx][k]) < 1e-4 * max(1.0, abs(grads[t_idx][k]))
