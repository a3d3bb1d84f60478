"""The batched-projection GEMM on the 5th-generation tensor cores
(csrc/nfb_umma.cu: tcgen05.mma + TMEM + TMA, stream-K with a deterministic
fixup) against the exact product: fp16 x fp16 products are exact in float64,
so the only error is the kernel's fp32 accumulation (~K * 2^-24 relative).
Shapes: every projection of the C4 bench (Pythia-2.8B, N = 2B hi/lo rows for
B = 1 / 4 / 16 / 64) plus ragged M / K / N edges."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def gemm(W, A):
    import torch
    from paper_2604_23553_b200 import _lib
    lib = _lib.load()
    M, K = W.shape
    N = A.shape[0]
    Wd = torch.from_numpy(W.astype(np.float16)).cuda()
    Ad = torch.from_numpy(A.astype(np.float16)).cuda()
    Y = torch.full((N, M), float("nan"), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.nfb_gemm_f16_dev(M, N, K, C.c_void_p(Wd.data_ptr()), C.c_void_p(Ad.data_ptr()),
                              C.c_void_p(Y.data_ptr()), C.c_void_p(st))
    assert rc == 0, rc
    torch.cuda.synchronize()
    return Y.cpu().numpy()


@pytest.mark.parametrize("M,N,K", [
    (7680, 2, 2560), (2560, 8, 2560), (10240, 32, 2560), (2560, 128, 10240), (50304, 8, 2560),
    (300, 24, 320), (128, 256, 64), (1000, 17, 72), (2560, 40, 10240),
])
def test_umma_gemm_matches_exact_product(M, N, K):
    rng = np.random.default_rng(M + 7 * N + K)
    W = (rng.uniform(-1, 1, (M, K)) / np.sqrt(K)).astype(np.float16)
    A = rng.standard_normal((N, K)).astype(np.float16)
    Y = gemm(W, A)
    want = A.astype(np.float64) @ W.astype(np.float64).T
    err = np.max(np.abs(Y - want)) / np.max(np.abs(want))
    assert np.isfinite(Y).all()
    assert err <= 4e-6, err


def test_umma_gemm_is_deterministic():
    rng = np.random.default_rng(3)
    W = (rng.uniform(-1, 1, (2560, 10240)) / 100).astype(np.float16)
    A = rng.standard_normal((128, 10240)).astype(np.float16)
    assert np.array_equal(gemm(W, A), gemm(W, A))


def test_preblocked_weights_entry_matches():
    """The steady-state entry (weights blocked once into the UMMA SW128 layout,
    csrc/nfb_umma.cuh) gives the same bits as block-then-run."""
    import torch
    from paper_2604_23553_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(11)
    M, N, K = 2560, 32, 10240
    W = (rng.uniform(-1, 1, (M, K)) / 100).astype(np.float16)
    A = rng.standard_normal((N, K)).astype(np.float16)
    Wd = torch.from_numpy(W).cuda()
    Ad = torch.from_numpy(A).cuda()
    Wb = torch.empty(lib.nfb_gemm_blocked_bytes(M, K) // 2, dtype=torch.float16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert lib.nfb_gemm_block_weights_dev(M, K, C.c_void_p(Wd.data_ptr()), C.c_void_p(Wb.data_ptr()),
                                          C.c_void_p(st)) == 0
    Y = torch.empty((N, M), dtype=torch.float32, device="cuda")
    assert lib.nfb_gemm_f16_blocked_dev(M, N, K, C.c_void_p(Wb.data_ptr()), C.c_void_p(Ad.data_ptr()),
                                        C.c_void_p(Y.data_ptr()), C.c_void_p(st)) == 0
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy(), gemm(W, A))
