"""tcgen05 / TMA GEMM kernel parity (every majorness, bf16 and 3xTF32).

bf16: compared with an fp32 torch product of the same bf16-rounded inputs,
tolerance 1e-3 relative (fp32 accumulation order only).  tf32 one segment:
against the torch product of tf32-truncated inputs.  3xTF32: against fp64,
tolerance 2e-6 relative (the fp32-accuracy claim of the fp32 mode).
"""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ptrs(ts):
    return (ctypes.c_void_p * 3)(*[t.data_ptr() for t in ts] + [0] * (3 - len(ts)))


def run_gemm(kind, a_mn, b_mn, bn, A_list, B_list, M, N, K, splits=1):
    from paper_2403_08837_b200 import _native

    L = _native.lib()
    dev = A_list[0].device
    D = torch.full((M, N), float("nan"), device=dev, dtype=torch.float32)
    ws = torch.empty(64 << 20, device=dev, dtype=torch.float32) if splits > 1 else None
    cnt = torch.zeros(4096, device=dev, dtype=torch.int32) if splits > 1 else None
    lda = A_list[0].shape[1]
    ldb = B_list[0].shape[1]
    rc = L.cdp_test_gemm(kind, a_mn, b_mn, bn, M, N, K, len(A_list), _ptrs(A_list), lda, _ptrs(B_list), ldb,
                         D.data_ptr(), N, splits, ws.data_ptr() if ws is not None else None,
                         cnt.data_ptr() if cnt is not None else None, None)
    _native.check(rc)
    torch.cuda.synchronize()
    return D


def make(kind, mn, M, N, K, dev, gen):
    """Logical A[M,K], B[K,N] plus their stored forms."""
    dt = torch.bfloat16 if kind == 0 else torch.float32
    pad = 8 if kind == 0 else 4
    A = torch.randn(M, K, generator=gen, device="cpu").to(dev)
    B = torch.randn(K, N, generator=gen, device="cpu").to(dev)
    a_mn, b_mn = mn

    def store(X, rows_first):  # rows_first: stored as X (row-major), else as X^T
        Y = X if rows_first else X.t()
        r, c = Y.shape
        cp = (c + pad - 1) // pad * pad
        S = torch.zeros(r, cp, device=dev, dtype=dt)
        S[:, :c] = Y.to(dt)
        return S

    # A K-major: A[m*lda+k] -> stored [M, K]; MN-major: stored [K, M]
    As = store(A, not a_mn)
    # B K-major: B[n*ldb+k] -> stored [N, K]; MN-major: stored [K, N]
    Bs = store(B, b_mn)
    return A.to(dt).float(), B.to(dt).float(), As, Bs


CASES = [
    # kind, (a_mn, b_mn), bn, M, N, K, splits
    (0, (0, 0), 32, 256, 32, 3072, 1),
    (0, (1, 0), 32, 256, 32, 3072, 1),
    (0, (1, 0), 32, 256, 32, 3072, 8),
    (0, (1, 1), 256, 3072, 256, 32, 1),
    (0, (1, 1), 64, 256, 10, 32, 1),
    (0, (0, 0), 32, 256, 32, 256, 1),
    (0, (0, 1), 128, 384, 256, 512, 1),
    (0, (0, 0), 256, 512, 512, 1024, 2),
    (0, (1, 0), 32, 10, 32, 256, 1),
    (1, (0, 0), 32, 256, 32, 512, 1),
    (1, (1, 0), 32, 256, 32, 3072, 4),
    (1, (1, 1), 256, 3072, 256, 32, 1),
    (1, (0, 1), 64, 256, 64, 256, 1),
    (1, (1, 1), 32, 256, 10, 32, 1),
]


@pytest.mark.parametrize("kind,mn,bn,M,N,K,splits", CASES)
def test_gemm_single_segment(cuda, kind, mn, bn, M, N, K, splits):
    gen = torch.Generator().manual_seed(M * 7 + N * 13 + K + kind)
    A, B, As, Bs = make(kind, mn, M, N, K, cuda, gen)
    D = run_gemm(kind, mn[0], mn[1], bn, [As], [Bs], M, N, K, splits)
    if kind == 1:  # tensor core reads tf32: compare against truncated operands
        def tf32(x):
            return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)
        ref = (tf32(A).double() @ tf32(B).double()).float()
        tol = 2e-3
    else:
        ref = (A.double() @ B.double()).float()
        tol = 1e-3
    err = (D - ref).abs().max().item() / (ref.abs().max().item() + 1e-30)
    assert err < tol, (err, D[:2, :4], ref[:2, :4])


@pytest.mark.parametrize("mn,bn,M,N,K,splits", [((1, 0), 32, 256, 32, 3072, 24), ((1, 1), 256, 3072, 256, 32, 1),
                                                ((0, 0), 32, 256, 32, 256, 1)])
def test_gemm_3xtf32_is_fp32_accurate(cuda, mn, bn, M, N, K, splits):
    """The tensor-core accumulator is not exact fp32 over long K, so the fp32
    mode keeps each TMEM accumulation to <= 256 of K (split-K, in-order fp32
    fix-up); with that the 3xTF32 product is within 1e-5 of fp64."""
    gen = torch.Generator().manual_seed(5)
    A = torch.randn(M, K, generator=gen).to(cuda)
    B = torch.randn(K, N, generator=gen).to(cuda)

    def split(X):
        hi = (X.view(torch.int32) & ~0x1FFF).view(torch.float32)
        return hi, X - hi

    def store(X, rows_first):
        Y = (X if rows_first else X.t()).contiguous()
        r, c = Y.shape
        cp = (c + 3) // 4 * 4
        S = torch.zeros(r, cp, device=cuda)
        S[:, :c] = Y
        return S

    Ah, Al = split(A)
    Bh, Bl = split(B)
    As = [store(Ah, not mn[0]), store(Ah, not mn[0]), store(Al, not mn[0])]
    Bs = [store(Bh, mn[1]), store(Bl, mn[1]), store(Bh, mn[1])]
    D = run_gemm(1, mn[0], mn[1], bn, As, Bs, M, N, K, splits)
    ref = A.double() @ B.double()
    err = ((D.double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-5, err
