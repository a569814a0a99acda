"""Register-spill guard for the persistent tcgen05 GEMM (CPU test: reads the built library's resource table).

A change in the epilogue once made every single-CTA gemm_pk_kernel spill 250-330 bytes of stack and cost
10-12 % of the ResNet / ViT step; this test fails when any bf16 gemm_pk_kernel instantiation uses more than
64 bytes of stack or any gemm_pk / pk_reduce kernel exceeds the register budget of its launch bounds.
"""
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2403_08837_b200",
                   "libcdp_b200.so")


def _resources():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(exe):
        pytest.skip("library or cuobjdump not available")
    out = subprocess.run([exe, "-res-usage", LIB], capture_output=True, text=True, timeout=300).stdout
    lines = out.splitlines()
    res = []
    for i, l in enumerate(lines):
        m = re.search(r"Function (\S+):", l)
        if m and i + 1 < len(lines):
            r = re.search(r"REG:(\d+) STACK:(\d+)", lines[i + 1])
            if r:
                res.append((m.group(1), int(r.group(1)), int(r.group(2))))
    return res


def test_gemm_pk_kernels_do_not_spill():
    res = [r for r in _resources() if "gemm_pk_kernel" in r[0]]
    assert res, "no gemm_pk_kernel in the library"
    # bf16 instantiations: mangled template argument list starts with Li0E (KIND = 0)
    bad = [(n, s) for n, _r, s in res if "gemm_pk_kernelILi0E" in n and s > 64]
    assert not bad, f"{len(bad)} bf16 gemm_pk_kernel instantiations use > 64 B of stack, e.g. {bad[:3]}"
    assert all(r <= 168 for _n, r, _s in res), "gemm_pk_kernel exceeds 168 registers (384-thread launch bound)"


def test_split_k_reduce_keeps_occupancy():
    """pk_reduce_kernel (256 threads) stays at <= 64 registers: the split-K tail is latency bound and
    needs its resident blocks (an epilogue change once took it to 80-96 registers)."""
    res = [r for r in _resources() if "pk_reduce_kernel" in r[0]]
    assert res, "no pk_reduce_kernel in the library"
    bad = [(n, r) for n, r, _s in res if r > 64]
    assert not bad, f"pk_reduce_kernel over 64 registers: {bad[:3]}"
