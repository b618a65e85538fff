"""GPU: the layer-plumbing kernels behind secure training, each against a
numpy restatement on random Z_2^w data (bit-exact): the one-launch Beaver
matrix-product reconstruction (every tile shape, split-K, narrow rings,
party 0 local or not), the limb GEMM's C-addend epilogue, column sums,
pooling window sums, bias-row adds, im2col / col2im."""

import numpy as np
import pytest
import torch

from oracle import train_sim as OT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2402_02320_b200 import kernels
    return kernels


def _rand(rng, shape, w):
    v = rng.integers(0, 1 << 63, size=shape, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=shape,
                                                                                              dtype=np.uint64)
    if w < 64:
        v &= np.uint64((1 << w) - 1)
    return v


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


def _mm(a, b):
    """u64 matmul mod 2^64 (numpy uint64 wraps)."""
    out = np.zeros((a.shape[0], b.shape[1]), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for k in range(a.shape[1]):
            out += np.outer(a[:, k], b[k, :])
    return out


@pytest.mark.parametrize("L,M,Kd,N,p0,w", [
    (3, 300, 25, 20, 0, 64),      # thin conv-like output: 128x32 tiles
    (3, 25, 4000, 20, 0, 64),     # tiny output, long K: split-K atomics
    (2, 130, 70, 130, 1, 64),     # 64x64 tiles
    (1, 77, 33, 9, -1, 64),       # party mode, party 0 not local
    (1, 77, 33, 9, 0, 64),
    (4, 50, 40, 16, 2, 32),       # narrow ring: no split
    (2, 3, 300, 5, 0, 64),
    (3, 1000, 30, 10, 0, 64),     # 128x10 tiles, partial k-tile
    (3, 2000, 25, 20, 1, 64),     # 128x20 tiles
    (2, 20, 3000, 10, 0, 64),     # 32x10 tiles, split-K
])
def test_beaver_gemm_matches_numpy(K, L, M, Kd, N, p0, w):
    rng = np.random.default_rng(M * 7 + N)
    D, E = _rand(rng, (M, Kd), w), _rand(rng, (Kd, N), w)
    A, B, C = _rand(rng, (L, M, Kd), w), _rand(rng, (L, Kd, N), w), _rand(rng, (L, M, N), w)
    Zd = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
    Cd, Ad, Bd = _dev(C), _dev(A), _dev(B)
    K.beaver_gemm(Zd, M * N, Cd.data_ptr(), M * N, _dev(D), _dev(E), Ad.data_ptr(), M * Kd, Bd.data_ptr(), Kd * N,
                  L, M, Kd, N, p0, w)
    got = _host(Zd)
    msk = np.uint64((1 << w) - 1) if w < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for l in range(L):
            Bl = B[l] + (E if l == p0 else np.uint64(0))
            want = (C[l] + _mm(D, Bl) + _mm(A[l], E)) & msk
            assert np.array_equal(got[l], want), l


def test_gemm_limbs_cin_epilogue(K):
    rng = np.random.default_rng(3)
    b, M, Kd, N = 2, 200, 96, 100
    A, B, C = _rand(rng, (b, M, Kd), 64), _rand(rng, (b, Kd, N), 64), _rand(rng, (b, M, N), 64)
    Mp, Np, Kp = K._rup(M, 128), K._rup(N, 64), K._rup(Kd, 128)
    Ad, Bd, Cd = _dev(A), _dev(B), _dev(C)
    for ks in (1, None):
        A8 = torch.zeros((b, 8, Mp, Kp), dtype=torch.uint8, device="cuda")
        B8 = torch.zeros((b, 8, Np, Kp), dtype=torch.uint8, device="cuda")
        for z in range(b):
            K.limb_split(A8[z], Ad.data_ptr() + 8 * z * M * Kd, M, Kd, Kd, Mp * Kp, Kp, 0, False)
            K.limb_split(B8[z], Bd.data_ptr() + 8 * z * Kd * N, Kd, N, N, Np * Kp, Kp, 0, True)
        Z = torch.full((b, M, N), 7, dtype=torch.int64, device="cuda")
        K.gemm_limbs(Z, A8, B8, b, M, N, Mp, Np, Kp, N, M * N, False, 64, ksplit=ks, cin=Cd, s_cin=M * N)
        got = _host(Z)
        with np.errstate(over="ignore"):
            for z in range(b):
                assert np.array_equal(got[z], C[z] + _mm(A[z], B[z]))


@pytest.mark.parametrize("L,rows,cols,w", [(3, 73728, 20, 64), (2, 1000, 500, 64), (1, 7, 3000, 32), (3, 5, 1, 64)])
def test_colsum(K, L, rows, cols, w):
    rng = np.random.default_rng(rows)
    x = _rand(rng, (L, rows, cols), w)
    out = torch.empty((L, cols), dtype=torch.int64, device="cuda")
    K.ring_colsum(out, _dev(x), L, rows, cols, w)
    with np.errstate(over="ignore"):
        want = x.sum(axis=1, dtype=np.uint64)
    if w < 64:
        want &= np.uint64((1 << w) - 1)
    assert np.array_equal(_host(out), want)


def test_pool_sum_and_add_rowvec(K):
    rng = np.random.default_rng(9)
    x = _rand(rng, (3, 4, 5, 24, 24), 64)
    out = torch.empty((3, 4, 5, 12, 12), dtype=torch.int64, device="cuda")
    K.ring_pool_sum(out, _dev(x), 60, 24, 24, 2, 64)
    with np.errstate(over="ignore"):
        want = x.reshape(3, 4, 5, 12, 2, 12, 2).sum(axis=(4, 6), dtype=np.uint64)
    assert np.array_equal(_host(out), want)
    z, b = _rand(rng, (3, 50, 20), 64), _rand(rng, (3, 20), 64)
    zd = _dev(z)
    K.ring_add_rowvec(zd, _dev(b), 3, 50, 20, 23, 64)
    with np.errstate(over="ignore"):
        want = z + (b << np.uint64(23))[:, None, :]
    assert np.array_equal(_host(zd), want)


@pytest.mark.parametrize("Bn,C,H,k,st,pd", [(4, 3, 12, 5, 1, 0), (2, 2, 9, 3, 2, 1), (3, 1, 28, 5, 1, 0)])
def test_im2col_col2im(K, Bn, C, H, k, st, pd):
    rng = np.random.default_rng(H)
    L = 2
    x = _rand(rng, (L, Bn, C, H, H), 64)
    OH = (H + 2 * pd - k) // st + 1
    cols = torch.empty((L, Bn * OH * OH, C * k * k), dtype=torch.int64, device="cuda")
    K.im2col(cols, _dev(x), L, Bn, C, H, H, k, st, pd)
    assert np.array_equal(_host(cols), OT.im2col(x, k, st, pd))
    g = _rand(rng, (L, Bn * OH * OH, C * k * k), 64)
    dx = torch.empty((L, Bn, C, H, H), dtype=torch.int64, device="cuda")
    K.col2im(dx, _dev(g), L, Bn, C, H, H, k, st, pd, 64)
    assert np.array_equal(_host(dx), OT.col2im(g, (L, Bn, C, H, H), k, st, pd, 64))


@pytest.mark.parametrize("M,Kd,N,b,mode", [(4000, 100, 640, 1, "cin"), (2048, 256, 300, 2, "acc"),
                                          (1500, 64, 1000, 1, "plain")])
def test_gemm_limbs_persistent_short_k(K, M, Kd, N, b, mode):
    """Short-K, many-tile products run on the persistent double-buffered
    tcgen05 kernel; exact vs numpy with each addend mode."""
    rng = np.random.default_rng(M + N)
    A, B, C = _rand(rng, (b, M, Kd), 64), _rand(rng, (b, Kd, N), 64), _rand(rng, (b, M, N), 64)
    Mp, Np, Kp = K._rup(M, 128), K._rup(N, 32), K._rup(Kd, 128)
    Ad, Bd, Cd = _dev(A), _dev(B), _dev(C)
    A8 = torch.zeros((b, 8, Mp, Kp), dtype=torch.uint8, device="cuda")
    B8 = torch.zeros((b, 8, Np, Kp), dtype=torch.uint8, device="cuda")
    for z in range(b):
        K.limb_split(A8[z], Ad.data_ptr() + 8 * z * M * Kd, M, Kd, Kd, Mp * Kp, Kp, 0, False)
        K.limb_split(B8[z], Bd.data_ptr() + 8 * z * Kd * N, Kd, N, N, Np * Kp, Kp, 0, True)
    Z = Cd.clone() if mode == "acc" else torch.full((b, M, N), 3, dtype=torch.int64, device="cuda")
    K.gemm_limbs(Z, A8, B8, b, M, N, Mp, Np, Kp, N, M * N, mode == "acc", 64, ksplit=1,
                 cin=Cd if mode == "cin" else None, s_cin=M * N)
    got = _host(Z)
    with np.errstate(over="ignore"):
        for z in range(b):
            want = _mm(A[z], B[z]) + (C[z] if mode in ("cin", "acc") else np.uint64(0))
            assert np.array_equal(got[z], want), z


@pytest.mark.parametrize("mode", ["cin", "acc", "plain"])
@pytest.mark.parametrize("ks", [1, 2, 3, None])
def test_gemm_limbs_persistent_splits(K, mode, ks):
    """Persistent tcgen05 kernel: every split-K slice count (wrapping atomics
    with the addend on slice 0, or onto the accumulate operand), an N tile
    that straddles Npad % 64 == 32, several units per CTA; exact vs numpy."""
    rng = np.random.default_rng(11 + (ks or 0))
    b, M, Kd, N = 2, 700, 300, 96
    A, B, C = _rand(rng, (b, M, Kd), 64), _rand(rng, (b, Kd, N), 64), _rand(rng, (b, M, N), 64)
    Mp, Np, Kp = K._rup(M, 128), K._rup(N, 32), K._rup(Kd, 128)
    Ad, Bd, Cd = _dev(A), _dev(B), _dev(C)
    A8 = torch.zeros((b, 8, Mp, Kp), dtype=torch.uint8, device="cuda")
    B8 = torch.zeros((b, 8, Np, Kp), dtype=torch.uint8, device="cuda")
    for z in range(b):
        K.limb_split(A8[z], Ad.data_ptr() + 8 * z * M * Kd, M, Kd, Kd, Mp * Kp, Kp, 0, False)
        K.limb_split(B8[z], Bd.data_ptr() + 8 * z * Kd * N, Kd, N, N, Np * Kp, Kp, 0, True)
    Z = Cd.clone() if mode == "acc" else torch.full((b, M, N), 5, dtype=torch.int64, device="cuda")
    K.gemm_limbs(Z, A8, B8, b, M, N, Mp, Np, Kp, N, M * N, mode == "acc", 64, ksplit=ks,
                 cin=Cd if mode == "cin" else None, s_cin=M * N)
    got = _host(Z)
    with np.errstate(over="ignore"):
        for z in range(b):
            want = _mm(A[z], B[z]) + (C[z] if mode in ("cin", "acc") else np.uint64(0))
            assert np.array_equal(got[z], want), z


@pytest.mark.parametrize("M,Kd,N,b", [(300, 20, 20, 3), (1000, 50, 30, 2), (700, 60, 100, 1), (256, 32, 64, 2),
                                      (130, 100, 20, 1)])
def test_gemm_limbs_short_k_blocks(K, M, Kd, N, b):
    """32- and 64-byte k-blocks (32B / 64B swizzle) and the 32-wide N tile of
    the persistent kernel; exact vs numpy with the C addend."""
    rng = np.random.default_rng(M + Kd + N)
    A, B, C = _rand(rng, (b, M, Kd), 64), _rand(rng, (b, Kd, N), 64), _rand(rng, (b, M, N), 64)
    Mp, Np, Kp = K._rup(M, 128), K._rup(N, 32), K.kpad(Kd)
    Ad, Bd, Cd = _dev(A), _dev(B), _dev(C)
    A8 = torch.zeros((b, 8, Mp, Kp), dtype=torch.uint8, device="cuda")
    B8 = torch.zeros((b, 8, Np, Kp), dtype=torch.uint8, device="cuda")
    for z in range(b):
        K.limb_split(A8[z], Ad.data_ptr() + 8 * z * M * Kd, M, Kd, Kd, Mp * Kp, Kp, 0, False)
        K.limb_split(B8[z], Bd.data_ptr() + 8 * z * Kd * N, Kd, N, N, Np * Kp, Kp, 0, True)
    Z = torch.full((b, M, N), 9, dtype=torch.int64, device="cuda")
    K.gemm_limbs(Z, A8, B8, b, M, N, Mp, Np, Kp, N, M * N, False, 64, cin=Cd, s_cin=M * N)
    got = _host(Z)
    with np.errstate(over="ignore"):
        for z in range(b):
            assert np.array_equal(got[z], C[z] + _mm(A[z], B[z])), z


@pytest.mark.parametrize("L,p0,jobs,m,k,r,xt,yt", [
    (3, 0, 1, 300, 130, 70, False, False),
    (2, 1, 2, 128, 64, 96, False, True),     # batched jobs, transposed B-side operand
    (3, 2, 1, 200, 25, 20, True, False),     # transposed A-side operand, 32-byte k-blocks, 32-wide N tile
    (4, 0, 3, 96, 200, 40, False, False),
])
def test_mask_limbs_split_gemm_matches_numpy(K, L, p0, jobs, m, k, r, xt, yt):
    """Fused sim-mode Beaver operands (mask + open + limb split, shared D/E
    limbs) and the split-operand GEMM: Z_l = C_l + D @ (B_l + [l==p0] E) +
    A_l @ E with D = sum_l X_l - A_l, E = sum_l Y_l - B_l (basic.py:66-75)."""
    rng = np.random.default_rng(m + k + r + jobs)
    X = _rand(rng, (jobs, L, m, k), 64)
    Y = _rand(rng, (jobs, L, k, r), 64)
    A, B, C = _rand(rng, (jobs, L, m, k), 64), _rand(rng, (jobs, L, k, r), 64), _rand(rng, (jobs, L, m, r), 64)
    # operands as the protocol sees them: [L, rows, cols] views (transposed storage when asked)
    Xd = _dev(np.ascontiguousarray(X.transpose(0, 1, 3, 2))).transpose(2, 3) if xt else _dev(X)
    Yd = _dev(np.ascontiguousarray(Y.transpose(0, 1, 3, 2))).transpose(2, 3) if yt else _dev(Y)
    Ad, Bd, Cd = _dev(A), _dev(B), _dev(C)
    Mp, Np, Kh = K._rup(m, 128), K._rup(r, 32), K.kpad(k)
    SA = torch.empty((jobs, 8, Mp, Kh), dtype=torch.uint8, device="cuda")
    PA = torch.empty((jobs, L, 8, Mp, Kh), dtype=torch.uint8, device="cuda")
    SB = torch.empty((jobs, 8, Np, Kh), dtype=torch.uint8, device="cuda")
    PB = torch.empty((jobs, L, 8, Np, Kh), dtype=torch.uint8, device="cuda")
    x0, y0 = Xd[0], Yd[0]
    K.mask_limbs(SA, PA, x0.data_ptr(), x0.stride(0), x0.stride(1), x0.stride(2), Ad.data_ptr(), m * k, k, 1, L, m,
                 k, Mp, Kh, p0, False, 64, jobs=jobs, x_js=Xd.stride(0), t_js=L * m * k)
    K.mask_limbs(SB, PB, y0.data_ptr(), y0.stride(0), y0.stride(2), y0.stride(1), Bd.data_ptr(), k * r, 1, r, L, r,
                 k, Np, Kh, p0, True, 64, jobs=jobs, x_js=Yd.stride(0), t_js=L * k * r)
    Z = torch.empty((jobs, L, m, r), dtype=torch.int64, device="cuda")
    K.gemm_limbs_split(Z, PA, SA, PB, SB, jobs * L, m, r, Mp, Np, Kh, r, m * r, 64, Cd.data_ptr(), m * r, zl=L,
                       s_cin_j=L * m * r)
    got = _host(Z)
    with np.errstate(over="ignore"):
        for j in range(jobs):
            D = (X[j] - A[j]).sum(0, dtype=np.uint64)
            E = (Y[j] - B[j]).sum(0, dtype=np.uint64)
            for l in range(L):
                Bl = B[j, l] + (E if l == p0 else np.uint64(0))
                want = C[j, l] + _mm(D, Bl) + _mm(A[j, l], E)
                assert np.array_equal(got[j, l], want), (j, l)


@pytest.mark.parametrize("L,p0,jobs,m,k,r,xt,yt", [
    (3, 0, 1, 300, 130, 70, False, False),
    (2, 1, 2, 128, 64, 96, False, True),
    (3, 2, 1, 200, 25, 20, True, False),
])
def test_mask_limbs2_matches_two_launches(K, L, p0, jobs, m, k, r, xt, yt):
    """Both operand sides in one launch write exactly the planes of the two
    per-side mask_limbs launches."""
    rng = np.random.default_rng(m * 3 + k + r + jobs)
    X, Y = _rand(rng, (jobs, L, m, k), 64), _rand(rng, (jobs, L, k, r), 64)
    A, B = _rand(rng, (jobs, L, m, k), 64), _rand(rng, (jobs, L, k, r), 64)
    Xd = _dev(np.ascontiguousarray(X.transpose(0, 1, 3, 2))).transpose(2, 3) if xt else _dev(X)
    Yd = _dev(np.ascontiguousarray(Y.transpose(0, 1, 3, 2))).transpose(2, 3) if yt else _dev(Y)
    Ad, Bd = _dev(A), _dev(B)
    Mp, Np, Kh = K._rup(m, 128), K._rup(r, 32), K.kpad(k)
    bufs = [torch.full(s, 7, dtype=torch.uint8, device="cuda") for s in
            [(jobs, 8, Mp, Kh), (jobs, L, 8, Mp, Kh), (jobs, 8, Np, Kh), (jobs, L, 8, Np, Kh)] * 2]
    x0, y0 = Xd[0], Yd[0]
    K.mask_limbs(bufs[0], bufs[1], x0.data_ptr(), x0.stride(0), x0.stride(1), x0.stride(2), Ad.data_ptr(), m * k, k,
                 1, L, m, k, Mp, Kh, p0, False, 64, jobs=jobs, x_js=Xd.stride(0), t_js=L * m * k)
    K.mask_limbs(bufs[2], bufs[3], y0.data_ptr(), y0.stride(0), y0.stride(2), y0.stride(1), Bd.data_ptr(), k * r, 1,
                 r, L, r, k, Np, Kh, p0, True, 64, jobs=jobs, x_js=Yd.stride(0), t_js=L * k * r)
    K.mask_limbs2(bufs[4], bufs[5], x0.data_ptr(), x0.stride(0), x0.stride(1), x0.stride(2), Ad.data_ptr(), m * k, k,
                  1, m, Mp, bufs[6], bufs[7], y0.data_ptr(), y0.stride(0), y0.stride(2), y0.stride(1), Bd.data_ptr(),
                  k * r, 1, r, r, Np, L, k, Kh, p0, 64, jobs=jobs, x_js=Xd.stride(0), a_js=L * m * k,
                  y_js=Yd.stride(0), b_js=L * k * r)
    for i in range(4):
        assert torch.equal(bufs[i], bufs[4 + i]), i


@pytest.mark.parametrize("L,p0,jobs,m,k,r,xt,yt,w", [
    (3, 0, 1, 25, 5000, 20, True, False, 64),    # conv weight gradient: tiny output, long K, X^T in place
    (3, 1, 1, 128, 500, 10, False, False, 64),   # thin FC output (128x10 tiles)
    (2, 0, 2, 500, 128, 10, True, False, 64),    # batched jobs
    (4, 3, 1, 128, 10, 500, False, True, 64),    # short K, transposed Y view, p0 = last party
    (3, 0, 1, 70, 33, 40, False, False, 32),     # narrow ring: no split
    (2, 1, 3, 20, 3000, 10, True, True, 64),
    # thin kernels: tall (huge M, K and N <= 32) and long-K (tiny output)
    (3, 0, 1, 9000, 25, 20, False, False, 64),   # LeNet conv1 forward shape family
    (2, 1, 2, 5000, 10, 16, False, True, 64),
    (4, 3, 1, 4100, 32, 32, True, False, 32),
    (3, 2, 1, 4096, 7, 5, False, False, 64),
    (3, 0, 1, 25, 73728, 20, True, False, 64),   # LeNet conv1 weight gradient at batch 128 (split-K tiles)
    (4, 1, 1, 10, 700, 9, False, True, 64),
])
@pytest.mark.parametrize("thin", ["1", "0"])
def test_beaver_gemm_sim_matches_numpy(K, monkeypatch, thin, L, p0, jobs, m, k, r, xt, yt, w):
    """Sim-mode Beaver opening + reconstruction in one launch: Z_l = C_l +
    D @ (B_l + [l==p0] E) + A_l @ E, D = sum_l X_l - A_l, E = sum_l Y_l - B_l
    (basic.py:66-75), mod 2^w - on the thin kernels (tall / long-K) where
    the shape fits them, and with them disabled (MPX_THIN=0: tiled kernel)."""
    monkeypatch.setenv("MPX_THIN", thin)
    rng = np.random.default_rng(m * 5 + k + r + jobs + w)
    X, Y = _rand(rng, (jobs, L, m, k), w), _rand(rng, (jobs, L, k, r), w)
    A, B, C = _rand(rng, (jobs, L, m, k), w), _rand(rng, (jobs, L, k, r), w), _rand(rng, (jobs, L, m, r), w)
    Xd = _dev(np.ascontiguousarray(X.transpose(0, 1, 3, 2))).transpose(2, 3) if xt else _dev(X)
    Yd = _dev(np.ascontiguousarray(Y.transpose(0, 1, 3, 2))).transpose(2, 3) if yt else _dev(Y)
    Ad, Bd, Cd = _dev(A), _dev(B), _dev(C)
    Z = torch.empty((jobs, L, m, r), dtype=torch.int64, device="cuda")
    x0, y0 = Xd[0], Yd[0]
    K.beaver_gemm_sim(Z, m * r, L * m * r, Cd.data_ptr(), m * r, L * m * r,
                      x0.data_ptr(), x0.stride(0), x0.stride(1), x0.stride(2), Xd.stride(0),
                      Ad.data_ptr(), m * k, L * m * k,
                      y0.data_ptr(), y0.stride(0), y0.stride(1), y0.stride(2), Yd.stride(0),
                      Bd.data_ptr(), k * r, L * k * r, L, jobs, m, k, r, p0, w)
    got = _host(Z)
    msk = np.uint64((1 << w) - 1) if w < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for j in range(jobs):
            D = (X[j] - A[j]).sum(0, dtype=np.uint64)
            E = (Y[j] - B[j]).sum(0, dtype=np.uint64)
            for l in range(L):
                Bl = B[j, l] + (E if l == p0 else np.uint64(0))
                want = (C[j, l] + _mm(D, Bl) + _mm(A[j, l], E)) & msk
                assert np.array_equal(got[j, l], want), (j, l)
