"""Thin sim-mode Beaver product on tcgen05 (mpx_beaver_tc_thin, limb operands
built in shared memory) vs a numpy u64 restatement of basic.py:66-75:
Z_l = C_l + D @ (B_l + [l == p0] E) + A_l @ E, D = sum X_l - A_l,
E = sum Y_l - B_l (mod 2^64), bit-exact. Shapes: LeNet conv1 forward
(73728 x 25 x 20, 3 parties) and ragged K / N / M at the kernel's limits,
X read through a transposed (strided) view."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

U = np.uint64


def _ref(X, A, Y, B, C, p0):
    D = (X.sum(0) - A.sum(0))
    E = (Y.sum(0) - B.sum(0))
    out = []
    with np.errstate(over="ignore"):
        for l in range(X.shape[0]):
            Bp = B[l] + (E if l == p0 else U(0))
            out.append(C[l] + _mm(D, Bp) + _mm(A[l], E))
    return np.stack(out)


def _mm(a, b):
    # exact u64 matmul mod 2^64 (numpy matmul on uint64 wraps)
    return np.matmul(a, b)


@pytest.mark.parametrize("L,M,K,N", [(3, 73728, 25, 20), (2, 1000, 32, 32), (3, 129, 1, 1), (3, 5000, 17, 9),
                                     (2, 4096, 31, 30)])
def test_thin_tc_matches_numpy(L, M, K, N):
    from paper_2402_02320_b200 import kernels as Kn
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    rnd = lambda *s: torch.randint(-2**63, 2**63 - 1, s, device="cuda", generator=g, dtype=torch.int64)  # noqa
    X, A, C = rnd(L, M, K), rnd(L, M, K), rnd(L, M, N)
    Y, B = rnd(L, K, N), rnd(L, K, N)
    Z = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
    Kn.beaver_tc_thin(Z, M * N, C.data_ptr(), M * N, X.data_ptr(), M * K, K, 1, A.data_ptr(), M * K,
                      Y.data_ptr(), K * N, N, 1, B.data_ptr(), K * N, L, M, K, N, 0, 64)
    torch.cuda.synchronize()
    f = lambda t: t.cpu().numpy().view(U)  # noqa: E731
    want = _ref(f(X), f(A), f(Y), f(B), f(C), 0)
    assert np.array_equal(f(Z), want)


def test_thin_tc_transposed_x_and_party1_constant():
    """X as a transposed view (column stride != 1) and p0 = 1."""
    from paper_2402_02320_b200 import kernels as Kn
    L, M, K, N = 3, 3000, 20, 12
    g = torch.Generator(device="cuda").manual_seed(5)
    rnd = lambda *s: torch.randint(-2**63, 2**63 - 1, s, device="cuda", generator=g, dtype=torch.int64)  # noqa
    XT = rnd(L, K, M)           # X = XT^T per party
    A, C, Y, B = rnd(L, M, K), rnd(L, M, N), rnd(L, K, N), rnd(L, K, N)
    Z = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
    Kn.beaver_tc_thin(Z, M * N, C.data_ptr(), M * N, XT.data_ptr(), K * M, 1, M, A.data_ptr(), M * K,
                      Y.data_ptr(), K * N, N, 1, B.data_ptr(), K * N, L, M, K, N, 1, 64)
    torch.cuda.synchronize()
    f = lambda t: t.cpu().numpy().view(U)  # noqa: E731
    X = np.ascontiguousarray(np.transpose(f(XT), (0, 2, 1)))
    assert np.array_equal(f(Z), _ref(X, f(A), f(Y), f(B), f(C), 1))
