"""Fused attention kernels (csrc/attn_kernels.cuh) against a plain PyTorch fp32 reference of the same op.

The ViT trainer's attention (north_star (4): ViT-B/16, T = 197 tokens, 12 heads of 64) runs as one fused
forward (S = Q K^T / 8 in TMEM, exact one-tile softmax, O = P V, row log-sum-exp) and one fused backward
(P recomputed from the log-sum-exp; dV, dP, dS, dQ, dK).  Inputs are bf16; the reference upcasts the
same bf16 values to fp32.  Tolerances (relative L2): the kernels round P and dS to bf16 before their
second GEMM, as the unfused path did, so O / dQ / dK / dV carry ~bf16 relative error.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_O = 1e-2
TOL_GRAD = 2e-2


def _rel(a, b):
    return float((a - b).norm() / b.norm())


def _run(torch, T, H, B, seed, pad=0):
    from paper_2403_08837_b200 import _native

    D = H * 64
    g = torch.Generator(device="cuda").manual_seed(seed)
    ld = 3 * D + pad
    qkv = (torch.randn(B * T, ld, device="cuda", generator=g) * 1.5).to(torch.bfloat16)
    dout = torch.randn(B * T, D + pad, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.zeros(B * T, D + pad, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(B * H * T, device="cuda", dtype=torch.float32)
    dqkv = torch.zeros(B * T, ld, device="cuda", dtype=torch.bfloat16)
    lib = _native.lib()
    _native.check(lib.cdp_attention(ctypes.c_void_p(qkv.data_ptr()), ld, ctypes.c_void_p(dout.data_ptr()), D + pad,
                                    T, H, B, ctypes.c_void_p(o.data_ptr()), D + pad, ctypes.c_void_p(lse.data_ptr()),
                                    ctypes.c_void_p(dqkv.data_ptr()), ld, 1))
    # fp32 reference on the same bf16 inputs
    x = qkv[:, :3 * D].float().view(B, T, 3, H, 64).permute(2, 0, 3, 1, 4)  # [3][B][H][T][64]
    q, k, v = (x[i].clone().requires_grad_(True) for i in range(3))
    s = q @ k.transpose(-1, -2) * 0.125
    p = torch.softmax(s, dim=-1)
    out = p @ v
    go = dout[:, :D].float().view(B, T, H, 64).permute(0, 2, 1, 3)
    out.backward(go)
    ref_lse = torch.logsumexp(s, dim=-1)  # [B][H][T]
    got_o = o[:, :D].float().view(B, T, H, 64).permute(0, 2, 1, 3)
    dx = dqkv[:, :3 * D].float().view(B, T, 3, H, 64).permute(2, 0, 3, 1, 4)
    return dict(o=(got_o, out.detach()), lse=(lse.view(B, H, T), ref_lse.detach()), dq=(dx[0], q.grad),
                dk=(dx[1], k.grad), dv=(dx[2], v.grad), pad=(dqkv[:, 3 * D:], o[:, D:]))


@pytest.mark.parametrize("T,H,B", [(197, 12, 2), (197, 2, 3), (64, 2, 2), (130, 1, 2), (256, 2, 1), (17, 3, 1)])
def test_fused_attention_matches_torch(cuda, T, H, B):
    import torch

    r = _run(torch, T, H, B, seed=T * 31 + H)
    assert _rel(*r["o"]) <= TOL_O, ("O", _rel(*r["o"]))
    assert float((r["lse"][0] - r["lse"][1]).abs().max()) <= 1e-3 * max(1.0, float(r["lse"][1].abs().max()))
    for name in ("dq", "dk", "dv"):
        assert _rel(*r[name]) <= TOL_GRAD, (name, _rel(*r[name]))


def test_fused_attention_leaves_padding_columns(cuda):
    """Rows are written only in their head's 64 columns (the ViT buffers carry a ones / pad column)."""
    import torch

    r = _run(torch, 197, 2, 2, seed=7, pad=16)
    dpad, opad = r["pad"]
    assert int(torch.count_nonzero(dpad)) == 0 and int(torch.count_nonzero(opad)) == 0
    assert _rel(*r["o"]) <= TOL_O and _rel(*r["dv"]) <= TOL_GRAD
