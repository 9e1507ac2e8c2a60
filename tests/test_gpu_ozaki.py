"""The Ozaki INT8 tensor-core GEMM (csrc/ozaki.cu: tcgen05.mma kind::i8 with
TMEM accumulators and TMA-fed SWIZZLE_32B tiles) against torch's fp64 GEMM.

Error model (ozaki.h): with s signed 7-bit slices per operand and per-row
scaling, every product term is exact except the truncated slice tails and
the dropped diagonals, so |C - C_ref| <= c * 2^(-7s) * max|A_m.| * max|B_n.| * K
with c a small constant; integer inputs that fit the slices are exact."""
import ctypes

import numpy as np
import pytest

from paper_2111_10105_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _oz(A, B, s, a_t=False, b_t=False):
    """C = A @ B.T through dmcg_ozaki_gemm.  a_t / b_t: pass the operand as
    the transpose of a stored matrix (row stride 1) to exercise both slicing
    layouts."""
    import torch
    M, K = A.shape
    N = B.shape[0]
    dA = (A.T.contiguous() if a_t else A.contiguous())
    dB = (B.T.contiguous() if b_t else B.contiguous())
    a_rs, a_ks = (1, M) if a_t else (K, 1)
    b_rs, b_ks = (1, N) if b_t else (K, 1)
    C = torch.empty((M, N), dtype=torch.float64, device="cuda")
    rc = L.lib().dmcg_ozaki_gemm(ctypes.c_void_p(dA.data_ptr()), int(A.dtype == torch.float32),
                                 a_rs, a_ks, M, ctypes.c_void_p(dB.data_ptr()),
                                 int(B.dtype == torch.float32), b_rs, b_ks, N, K, s,
                                 ctypes.c_void_p(C.data_ptr()))
    assert rc == 0
    return C


@pytest.mark.parametrize("M,N,K,dtype,s,a_t,b_t", [
    (128, 64, 32, "f64", 7, False, False),
    (200, 100, 300, "f64", 7, False, False),
    (200, 100, 300, "f64", 5, True, False),
    (256, 130, 1000, "f32", 5, False, True),
    (512, 512, 40000, "f32", 5, True, True),     # Gram-shaped: K = vertices, split-K
    (96, 257, 513, "f64", 6, True, True),
])
def test_ozaki_matches_fp64_gemm(M, N, K, dtype, s, a_t, b_t):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    A = torch.randn((M, K), generator=g, device="cuda", dtype=torch.float64).to(tdt)
    B = torch.randn((N, K), generator=g, device="cuda", dtype=torch.float64).to(tdt)
    A[:, :7] *= 1e-3     # rows with mixed magnitudes
    C = _oz(A, B, s, a_t, b_t)
    ref = A.double() @ B.double().T
    bound = 8.0 * 2.0 ** (-7 * s) * A.abs().amax(1, keepdim=True).double() * \
        B.abs().amax(1).double()[None, :] * K
    err = (C - ref).abs()
    assert bool((err <= bound).all()), float((err / bound).max())


def test_ozaki_exact_on_small_integers():
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randint(-1000, 1000, (300, 777), generator=g, device="cuda").double()
    B = torch.randint(-1000, 1000, (190, 777), generator=g, device="cuda").double()
    C = _oz(A, B, 3)        # |x| < 2^10: two balanced digits represent it exactly
    assert torch.equal(C, A @ B.T)


def test_ozaki_gram_symmetric_and_rank_one():
    """X^T X of a rank-1, time-invariant axis (c3's x / y axes): exactly
    symmetric (the slice-pair set is symmetric) and equal to the fp64 Gram."""
    import torch
    n, F = 5000, 64
    x = torch.linspace(0, 1, n, device="cuda", dtype=torch.float32)
    X = x[:, None].repeat(1, F)            # n x F, every frame the same
    Xt = X.T.contiguous()                  # F x n: rows = frames, K = vertices
    C = _oz(Xt, Xt, 5)
    assert torch.equal(C, C.T)
    ref = Xt.double() @ Xt.double().T
    assert float(((C - ref).abs() / ref.abs().max()).max()) < 1e-11
