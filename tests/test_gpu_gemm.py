"""K3 tcgen05 TF32 GEMM vs a float64 NumPy product (TF32 inputs, fp32 accumulate:
normwise relative error well inside the north star's 2e-3)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_02300_b200 import gnnpart as gp
    return gp.Context(0)


def gemm(ctx, A, B, split=1, precision=1):
    from paper_2404_02300_b200._lib import check, lib
    A = np.ascontiguousarray(A, np.float32); B = np.ascontiguousarray(B, np.float32)
    M, K = A.shape; N = B.shape[0]
    out = np.zeros((M, N), np.float32)
    check(lib.catgnn_gemm_tn(ctx.handle, M, N, K, A.ctypes.data_as(C.c_void_p), B.ctypes.data_as(C.c_void_p),
                             out.ctypes.data_as(C.c_void_p), split, precision))
    return out


@pytest.mark.parametrize("M,N,K,split", [(128, 16, 32, 1), (1, 16, 8, 1), (200, 48, 256, 1), (1000, 256, 602, 1),
                                         (300, 602, 256, 1), (48, 256, 5000, 0), (256, 602, 20000, 0),
                                         (513, 41, 100, 1), (130, 128, 64, 3),
                                         # CTA-pair (cta_group::2) tiles: M >= 256, row/column tails
                                         (256, 16, 8, 1), (4096, 256, 604, 1), (2000, 48, 256, 1),
                                         (777, 100, 48, 1), (1100, 602, 256, 1), (3000, 256, 1000, 4)])
def test_gemm_tn(ctx, M, N, K, split):
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    got = gemm(ctx, A, B, split)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 1e-3, err
    got3 = gemm(ctx, A, B, split, precision=3)
    err3 = np.linalg.norm(got3 - want) / np.linalg.norm(want)
    assert err3 < 2e-5, err3


def test_gemm_cancellation_needs_3xtf32(ctx):
    # weight-gradient shape: long K with heavy cancellation (result << terms)
    rng = np.random.default_rng(11)
    A = rng.standard_normal((64, 20000)).astype(np.float32)
    B = rng.standard_normal((96, 20000)).astype(np.float32)
    B[:, 10000:] = -B[:, :10000] * np.float32(0.999)
    A[:, 10000:] = A[:, :10000]
    want = A.astype(np.float64) @ B.astype(np.float64).T   # ~1000x smaller than its terms
    err1 = np.linalg.norm(gemm(ctx, A, B, 0, 1) - want) / np.linalg.norm(want)
    err3 = np.linalg.norm(gemm(ctx, A, B, 0, 3) - want) / np.linalg.norm(want)
    assert err3 < err1 / 50 and err3 < 1e-2, (err1, err3)


def gemm_general(ctx, A, a_mn, B, b_mn, split=1, precision=1):
    """A: M x K (a_mn=0) or K x M (a_mn=1); B: N x K or K x N."""
    from paper_2404_02300_b200._lib import check, lib
    A = np.ascontiguousarray(A, np.float32); B = np.ascontiguousarray(B, np.float32)
    M = A.shape[1] if a_mn else A.shape[0]
    K = A.shape[0] if a_mn else A.shape[1]
    N = B.shape[1] if b_mn else B.shape[0]
    out = np.zeros((M, N), np.float32)
    check(lib.catgnn_gemm(ctx.handle, M, N, K, A.ctypes.data_as(C.c_void_p), int(a_mn),
                          B.ctypes.data_as(C.c_void_p), int(b_mn), out.ctypes.data_as(C.c_void_p), split, precision))
    return out


@pytest.mark.parametrize("a_mn,b_mn", [(1, 1), (1, 0), (0, 1)])
@pytest.mark.parametrize("M,N,K,split,prec", [(256, 604, 20000, 0, 3), (41, 256, 3000, 0, 1), (41, 256, 3000, 0, 3),
                                              (128, 96, 64, 1, 1), (300, 33, 100, 1, 3), (16, 602, 999, 0, 1),
                                              (1024, 256, 700, 1, 3), (600, 130, 96, 1, 1)])
def test_gemm_mn_major(ctx, a_mn, b_mn, M, N, K, split, prec):
    """Weight-gradient form C = X^T Y read from row-major activations (no transpose)."""
    rng = np.random.default_rng(M + 3 * N + K)
    A = rng.standard_normal((K, M) if a_mn else (M, K)).astype(np.float32)
    B = rng.standard_normal((K, N) if b_mn else (N, K)).astype(np.float32)
    Al = A.T if a_mn else A
    Bl = B.T if b_mn else B
    want = Al.astype(np.float64) @ Bl.astype(np.float64).T
    got = gemm_general(ctx, A, a_mn, B, b_mn, split, prec)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < (2e-5 if prec == 3 else 1e-3), err


def test_gemm_k_zero(ctx):
    A = np.zeros((5, 0), np.float32); B = np.zeros((16, 0), np.float32)
    assert np.all(gemm(ctx, A, B) == 0)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 1), (0, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K,split", [(200, 48, 256, 1), (4096, 256, 604, 1), (256, 604, 20000, 0),
                                         (41, 256, 3000, 0), (2000, 256, 41, 1), (513, 41, 100, 1),
                                         (1100, 602, 256, 1), (3000, 256, 1000, 4), (128, 16, 64, 1),
                                         (777, 130, 200, 1)])
def test_gemm_bf16x3(ctx, a_mn, b_mn, M, N, K, split):
    """bf16x3 path (pre-split hi/lo operands, kind::f16 MMAs, no conversion pass):
    every operand layout the GNN uses, tails in M / N / K, split-K and CTA pairs."""
    rng = np.random.default_rng(M * 5 + N * 3 + K + 7 * a_mn + 11 * b_mn)
    A = rng.standard_normal((K, M) if a_mn else (M, K)).astype(np.float32)
    B = rng.standard_normal((K, N) if b_mn else (N, K)).astype(np.float32)
    Al = A.T if a_mn else A
    Bl = B.T if b_mn else B
    want = Al.astype(np.float64) @ Bl.astype(np.float64).T
    got = gemm_general(ctx, A, a_mn, B, b_mn, split, 4)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 5e-5, err


def test_gemm_bf16x3_cancellation(ctx):
    # the weight-gradient cancellation case: bf16x3 stays ~1e-4 of the (1000x smaller) result
    rng = np.random.default_rng(11)
    A = rng.standard_normal((64, 20000)).astype(np.float32)
    B = rng.standard_normal((96, 20000)).astype(np.float32)
    B[:, 10000:] = -B[:, :10000] * np.float32(0.999)
    A[:, 10000:] = A[:, :10000]
    want = A.astype(np.float64) @ B.astype(np.float64).T
    err1 = np.linalg.norm(gemm(ctx, A, B, 0, 1) - want) / np.linalg.norm(want)
    err4 = np.linalg.norm(gemm_general(ctx, A, 0, B, 0, 0, 4) - want) / np.linalg.norm(want)
    assert err4 < err1 / 20 and err4 < 2e-2, (err1, err4)
