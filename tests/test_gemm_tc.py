"""GPU: the tcgen05 int8-limb Z_2^64 GEMM against exact uint64 products.

numpy's uint64 matmul wraps mod 2^64 (the reference's ring.matmul,
ring.py:60-62), so it is the oracle here. Covers ragged shapes (padding),
the all-0xFF worst case for the per-diagonal s32 accumulators at K = 16384
(the bound the kernel relies on), K > 16384 chunking, batching with a
broadcast operand, accumulate-into-C and narrow widths.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _run(A, B, batch=1, sA=None, sB=None, acc=None, width=64):
    from paper_2402_02320_b200 import kernels as K
    M, Kd = A.shape[-2:]
    N = B.shape[-1]
    C = torch.zeros((batch, M, N), dtype=torch.int64, device="cuda")
    if acc is not None:
        C.copy_(_dev(acc))
    K.gemm_tc(C, _dev(A), _dev(B), batch, M, Kd, N, M * Kd if sA is None else sA,
              Kd * N if sB is None else sB, M * N, acc is not None, width)
    torch.cuda.synchronize()
    return _host(C)


@pytest.mark.parametrize("M,K,N", [(128, 128, 64), (200, 300, 100), (256, 384, 192), (1000, 513, 77),
                                   (512, 4096, 256)])
def test_random_shapes_exact(M, K, N):
    rng = np.random.default_rng(M * 7 + K * 3 + N)
    A = rng.integers(0, 1 << 64, (M, K), dtype=np.uint64)
    B = rng.integers(0, 1 << 64, (K, N), dtype=np.uint64)
    got = _run(A, B)[0]
    assert np.array_equal(got, np.matmul(A, B))


def test_all_ones_worst_case_k16384():
    M, K, N = 128, 16384, 64
    A = np.full((M, K), np.uint64(0xFFFFFFFFFFFFFFFF))
    B = np.full((K, N), np.uint64(0xFFFFFFFFFFFFFFFF))
    got = _run(A, B)[0]
    want = np.full((M, N), np.uint64((K * ((1 << 64) - 1) ** 2) % (1 << 64)))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("M,K,N", [(25, 147456, 20), (500, 16384, 50), (128, 40000, 10), (8, 3000, 700)])
def test_split_k_skinny_shapes(M, K, N):
    """conv-backward shapes: tiny M or N with long K, split-K atomics mod 2^64"""
    rng = np.random.default_rng(M + K + N)
    A = rng.integers(0, 1 << 64, (M, K), dtype=np.uint64)
    B = rng.integers(0, 1 << 64, (K, N), dtype=np.uint64)
    C0 = rng.integers(0, 1 << 64, (1, M, N), dtype=np.uint64)
    assert np.array_equal(_run(A, B)[0], np.matmul(A, B))
    assert np.array_equal(_run(A, B, acc=C0)[0], C0[0] + np.matmul(A, B))


def test_k_chunking_beyond_16384():
    rng = np.random.default_rng(3)
    A = rng.integers(0, 1 << 64, (128, 20000), dtype=np.uint64)
    B = rng.integers(0, 1 << 64, (20000, 64), dtype=np.uint64)
    assert np.array_equal(_run(A, B)[0], np.matmul(A, B))


def test_batched_broadcast_accumulate_width32():
    rng = np.random.default_rng(4)
    M, K, N, b = 192, 256, 128, 3
    A = rng.integers(0, 1 << 64, (M, K), dtype=np.uint64)          # broadcast (sA = 0)
    B = rng.integers(0, 1 << 64, (b, K, N), dtype=np.uint64)
    C0 = rng.integers(0, 1 << 64, (b, M, N), dtype=np.uint64)
    got = _run(A, B, batch=b, sA=0, acc=C0, width=32)
    want = (C0 + np.matmul(A[None], B)) & np.uint64(0xFFFFFFFF)
    assert np.array_equal(got, want)


def test_tc_matches_simt_path():
    from paper_2402_02320_b200 import kernels as K
    rng = np.random.default_rng(5)
    M, Kd, N = 256, 640, 192
    A = rng.integers(0, 1 << 64, (M, Kd), dtype=np.uint64)
    B = rng.integers(0, 1 << 64, (Kd, N), dtype=np.uint64)
    C1 = torch.empty((M, N), dtype=torch.int64, device="cuda")
    C2 = torch.empty((M, N), dtype=torch.int64, device="cuda")
    K.gemm_tc(C1, _dev(A), _dev(B), 1, M, Kd, N, 0, 0, 0, False, 64)
    K.gemm(C2, _dev(A), _dev(B), 1, M, Kd, N, 0, 0, 0, False, 64, simt=True)
    assert torch.equal(C1, C2)


@pytest.mark.parametrize("M,K,N,acc", [(128, 500, 10, False), (500, 128, 10, True), (3, 4000, 7, False),
                                       (200, 300, 100, True)])
def test_simt_split_k_exact(M, K, N, acc):
    from paper_2402_02320_b200 import kernels as K_
    rng = np.random.default_rng(M * K + N)
    A = rng.integers(0, 1 << 64, (M, K), dtype=np.uint64)
    B = rng.integers(0, 1 << 64, (K, N), dtype=np.uint64)
    C0 = rng.integers(0, 1 << 64, (M, N), dtype=np.uint64)
    C = _dev(C0) if acc else torch.zeros((M, N), dtype=torch.int64, device="cuda")
    K_.gemm(C, _dev(A), _dev(B), 1, M, K, N, 0, 0, 0, acc, 64, simt=True)
    torch.cuda.synchronize()
    want = np.matmul(A, B) + (C0 if acc else np.uint64(0))
    assert np.array_equal(_host(C), want)
