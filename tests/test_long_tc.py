"""Long-K sim-mode Beaver product on tcgen05 (mpx_beaver_tc_long: split-K over
the SMs, party-stacked limb MMAs, atomic split-K sum) vs a numpy u64
restatement of basic.py:66-75: Z_l = C_l + D @ (B_l + [l == p0] E) + A_l @ E,
D = sum X_l - A_l, E = sum Y_l - B_l (mod 2^64), bit-exact. Shapes: LeNet
conv1 weight gradient (cols^T @ dZ: 25 x 73728 x 20 at three parties, X a
transposed view) and ragged M / N / K at the kernel's limits, including a K
long enough that a CTA's range hits the 512-block exactness cap."""
import numpy as np
import pytest
import torch

from test_thin_tc import _ref

pytestmark = pytest.mark.gpu

U = np.uint64


def _run(L, M, K, N, p0, xt, seed):
    from paper_2402_02320_b200 import kernels as Kn
    g = torch.Generator(device="cuda").manual_seed(seed)
    rnd = lambda *s: torch.randint(-2**63, 2**63 - 1, s, device="cuda", generator=g, dtype=torch.int64)  # noqa
    A, C, Y, B = rnd(L, M, K), rnd(L, M, N), rnd(L, K, N), rnd(L, K, N)
    f = lambda t: t.cpu().numpy().view(U)  # noqa: E731
    if xt:   # X = XT^T per party (the transposed im2col view)
        XT = rnd(L, K, M)
        xp, xs = (XT.data_ptr(), K * M, 1, M), np.ascontiguousarray(np.transpose(f(XT), (0, 2, 1)))
    else:
        X = rnd(L, M, K)
        xp, xs = (X.data_ptr(), M * K, K, 1), f(X)
    Z = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
    assert Kn.long_tc_ok(L, M, K, N, 64)
    Kn.beaver_tc_long(Z, M * N, C.data_ptr(), M * N, *xp, A.data_ptr(), M * K,
                      Y.data_ptr(), K * N, N, 1, B.data_ptr(), K * N, L, M, K, N, p0, 64)
    torch.cuda.synchronize()
    return f(Z), _ref(xs, f(A), f(Y), f(B), f(C), p0)


@pytest.mark.parametrize("L,M,K,N,p0,xt", [(3, 25, 73728, 20, 0, True), (2, 32, 5000, 32, 1, False),
                                           (3, 1, 33, 1, 2, False), (3, 17, 4097, 9, 0, True),
                                           (2, 20, 100, 25, -1, True)])
def test_long_tc_matches_numpy(L, M, K, N, p0, xt):
    got, want = _run(L, M, K, N, p0, xt, M * 7 + K + N)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("env", ["MPX_LONG_ROW8", "MPX_LONG_NO_TMAP"])
def test_long_tc_fill_paths(monkeypatch, env):
    """MPX_LONG_ROW8=1: every family through the one-word-per-copy fill;
    MPX_LONG_NO_TMAP=1: the material rows by 256-byte bulk copies instead of
    the tensor-map boxes."""
    monkeypatch.setenv(env, "1")
    got, want = _run(3, 25, 3000, 20, 0, True, 3)
    assert np.array_equal(got, want)


def test_long_tc_exactness_cap():
    """K = 148 x 600 blocks: more than 512 k-blocks per SM, so the kernel
    launches more CTAs than SMs and every diagonal accumulator stays exact."""
    got, want = _run(2, 4, 148 * 600 * 32, 3, 0, False, 11)
    assert np.array_equal(got, want)


def test_long_tc_limits():
    from paper_2402_02320_b200 import kernels as Kn
    assert not Kn.long_tc_ok(3, 33, 1000, 20, 64)
    assert not Kn.long_tc_ok(3, 25, 1000, 20, 32)
    assert not Kn.long_tc_ok(4, 25, 1000, 20, 64)
    assert not Kn.long_tc_ok(3, 32, 1000, 32, 64)     # shared-memory budget at three parties
    assert Kn.long_tc_ok(2, 32, 1000, 32, 64)
