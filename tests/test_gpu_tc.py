"""GPU: the tcgen05 primitives (tc.cuh) through the test-only one-CTA TF32 GEMM export."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def core_off(r, k, Kc):
    return (r // 8) * (Kc * 32) + (k // 4) * 128 + (r % 8) * 16 + (k % 4) * 4


def tf32(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)     # round-half-away on the 13 dropped bits
    return u.view(np.float32)


def image(B):
    N, K = B.shape
    hi = tf32(B)
    lo = tf32(B - hi)
    img = np.zeros(2 * N * K, np.float32)
    for r in range(N):
        for k in range(K):
            o = core_off(r, k, K) // 4
            img[o] = hi[r, k]
            img[N * K + o] = lo[r, k]
    return img


@pytest.mark.parametrize("N,K", [(16, 8), (64, 40), (128, 72), (256, 32)])
def test_tc_gemm(N, K):
    from paper_2602_11896_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(N * 1000 + K)
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    Ad = torch.from_numpy(A).cuda()
    Bd = torch.from_numpy(image(B)).cuda()
    for three, tol in ((0, 3e-3), (1, 2e-6)):
        D = torch.zeros(128, N, device="cuda")
        _lib.check(lib.jtfs_debug_tc_gemm(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), N, K, three,
                                          torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        err = np.abs(D.cpu().numpy() - ref).max() / np.abs(ref).max()
        assert err < tol, (three, err)


@pytest.mark.parametrize("N,K", [(16, 16), (64, 64), (128, 128), (256, 32)])
def test_tc_gemm_a_in_tmem(N, K):
    from paper_2602_11896_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(N * 7 + K)
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    Ad = torch.from_numpy(A).cuda()
    Bd = torch.from_numpy(image(B)).cuda()
    for three, tol in ((0, 3e-3), (1, 2e-6)):
        D = torch.zeros(128, N, device="cuda")
        _lib.check(lib.jtfs_debug_tc_gemm_ts(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), N, K, three,
                                             torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        err = np.abs(D.cpu().numpy() - ref).max() / np.abs(ref).max()
        assert err < tol, (three, err)
