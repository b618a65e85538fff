"""Typed launch wrappers over the libmpx C ABI (one per entry point).

Every wrapper takes torch int64 tensors (uint64 words) already laid out as
include/mpx.h describes, skips the launch when its output is a ``meta``
tensor (dry run), and raises ``MpxError`` on failure.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from ._lib import call, ptr

_M64 = (1 << 64) - 1


def _u(v: int) -> int:
    return int(v) & _M64


def _dry(*ts) -> bool:
    return _lib.is_dry(*ts)


# ---- local ring ----------------------------------------------------------

def ring_lin(out, a, ka, b, kb, c0, cv, L, n, width, p0):
    if _dry(out):
        return out
    call("mpx_ring_lin", ptr(out), ptr(a), _u(ka), ptr(b), _u(kb), _u(c0), ptr(cv),
         int(cv.numel()) if cv is not None else 0, L, n, width, p0)
    return out


def ring_mul(out, a, b, n, width):
    if _dry(out):
        return out
    call("mpx_ring_mul", ptr(out), ptr(a), ptr(b), n, width)
    return out


def ring_rowdot(out, x, wts, L, rows, cols, width):
    if _dry(out):
        return out
    call("mpx_ring_rowdot", ptr(out), ptr(x), ptr(wts), L, rows, cols, width)
    return out


def encode(out, x_f64, n, width, frac):
    if _dry(out):
        return out
    call("mpx_encode", ptr(out), ptr(x_f64), n, width, frac)
    return out


def decode(out_f64, x, n, width, frac):
    if _dry(out_f64):
        return out_f64
    call("mpx_decode", ptr(out_f64), ptr(x), n, width, frac)
    return out_f64


def to_signed(out, x, n, width):
    if _dry(out):
        return out
    call("mpx_to_signed", ptr(out), ptr(x), n, width)
    return out


# ---- openings ------------------------------------------------------------

def open_sum(out, x, L, n, width):
    if _dry(out):
        return out
    call("mpx_open_sum", ptr(out), ptr(x), L, n, width)
    return out


def open_xor(out, x, L, n):
    if _dry(out):
        return out
    call("mpx_open_xor", ptr(out), ptr(x), L, n)
    return out


def mask_sub(out, x, a_ptr, a_ps, L, n, width):
    if _dry(out):
        return out
    call("mpx_mask_sub", ptr(out), ptr(x), a_ptr, a_ps, L, n, width)
    return out


class TruncJob(ctypes.Structure):
    _fields_ = [("z", ctypes.c_void_p), ("base", ctypes.c_void_p), ("x", ctypes.c_void_p),
                ("r_lo", ctypes.c_void_p), ("r_hi", ctypes.c_void_p), ("lo_ps", ctypes.c_int64),
                ("hi_ps", ctypes.c_int64), ("n", ctypes.c_int64), ("bias", ctypes.c_uint64),
                ("unbias", ctypes.c_uint64), ("f", ctypes.c_int), ("pad", ctypes.c_int)]


TRUNC_JOBS_MAX = 16


class TruncJobs(ctypes.Structure):
    _fields_ = [("j", TruncJob * TRUNC_JOBS_MAX), ("start", ctypes.c_int64 * (TRUNC_JOBS_MAX + 1)),
                ("n", ctypes.c_int), ("pad", ctypes.c_int)]


def trunc_sub_multi(jobs, L, width, p0):
    """jobs: list of dicts z, base (or None), x, r_lo, lo_ps, r_hi (or None), hi_ps, n, f, bias, unbias."""
    if not jobs or _dry(jobs[0]["z"]):
        return
    J = TruncJobs()
    J.n = len(jobs)
    for i, jb in enumerate(jobs):
        t = J.j[i]
        t.z, t.x = ptr(jb["z"]), ptr(jb["x"])
        t.base = ptr(jb["base"]) if jb["base"] is not None else None
        t.r_lo, t.r_hi = jb["r_lo"], jb["r_hi"]
        t.lo_ps, t.hi_ps, t.n = jb["lo_ps"], jb["hi_ps"], jb["n"]
        t.bias, t.unbias, t.f = jb["bias"], jb["unbias"], jb["f"]
    call("mpx_trunc_sub_multi", ctypes.addressof(J), L, width, p0)


def trunc_rows_bias(z, x, brow, bshift, r_lo, lo_ps, r_hi, hi_ps, L, B, S, C, nchw, width, f, bias, unbias, p0):
    if _dry(z):
        return z
    call("mpx_trunc_rows_bias", ptr(z), ptr(x), ptr(brow) if brow is not None else None, bshift, r_lo, lo_ps,
         r_hi, hi_ps, L, B, S, C, int(nchw), width, f, bias, unbias, p0)
    return z


def trunc_expand_rows(z, x, r_lo, lo_ps, r_hi, hi_ps, L, B, C, Hs, Ws, k, width, f, bias, unbias, p0):
    if _dry(z):
        return z
    call("mpx_trunc_expand_rows", ptr(z), ptr(x), r_lo, lo_ps, r_hi, hi_ps, L, B, C, Hs, Ws, k, width, f, bias,
         unbias, p0)
    return z


def mask_sub_t(out, x_ptr, x_ps, a_ptr, a_ps, L, rows, cols, width, batch=1, x_bs=0, a_bs=0):
    if _dry(out):
        return out
    call("mpx_mask_sub_t", ptr(out), x_ptr, x_ps, x_bs, a_ptr, a_ps, a_bs, L, batch, rows, cols, width)
    return out


def mask_sub_bs(out, x_ptr, x_ps, x_bs, a_ptr, a_ps, a_bs, L, batch, n, width):
    if _dry(out):
        return out
    call("mpx_mask_sub_bs", ptr(out), x_ptr, x_ps, x_bs, a_ptr, a_ps, a_bs, L, batch, n, width)
    return out


def transposed_base(v):
    """Party stride when ``v`` [L, r, c] is the last-two-axes transpose of a
    [c, r]-contiguous matrix per party (any party stride), else None."""
    if v.dim() != 3 or v.is_contiguous():
        return None
    L, r, c = v.shape
    if v.stride(1) == 1 and v.stride(2) == r and (L == 1 or v.stride(0) >= r * c):
        return v.stride(0)
    return None


def rows_base(v):
    """Party stride when ``v`` [L, ...] is row-major contiguous within each
    party (any party stride), else None."""
    if v.dim() < 2:
        return None
    inner = v[0] if v.shape[0] > 0 else v
    n = inner.numel()
    if inner.is_contiguous() and (v.shape[0] == 1 or v.stride(0) >= n):
        return v.stride(0)
    return None


# ---- Beaver arithmetic ----------------------------------------------------

def mul_finish(z, d, e, a, b, c, t_ps, L, n, width, p0):
    if _dry(z):
        return z
    call("mpx_mul_finish", ptr(z), ptr(d), ptr(e), a, b, c, t_ps, L, n, width, p0)
    return z


def mul_fused(z, x, y, a, b, c, t_ps, L, n, width, p0):
    if _dry(z):
        return z
    call("mpx_mul_fused", ptr(z), ptr(x), ptr(y), a, b, c, t_ps, L, n, width, p0)
    return z


def trunc_mask(out, x, r_lo, lo_ps, r_hi, hi_ps, L, n, width, f, bias, p0):
    if _dry(out):
        return out
    call("mpx_trunc_mask", ptr(out), ptr(x), r_lo, lo_ps, r_hi, hi_ps, L, n, width, f, _u(bias), p0)
    return out


def trunc_finish(z, c, r_hi, hi_ps, L, n, width, f, unbias, p0):
    if _dry(z):
        return z
    call("mpx_trunc_finish", ptr(z), ptr(c), r_hi, hi_ps, L, n, width, f, _u(unbias), p0)
    return z


def trunc_fused(z, x, r_lo, lo_ps, r_hi, hi_ps, L, n, width, f, bias, unbias, p0):
    if _dry(z):
        return z
    call("mpx_trunc_fused", ptr(z), ptr(x), r_lo, lo_ps, r_hi, hi_ps, L, n, width, f, _u(bias),
         _u(unbias), p0)
    return z


# ---- binary circuits -------------------------------------------------------

def and_mask(d, e, x, y, t, L, rows, m):
    if _dry(d):
        return
    call("mpx_and_mask", ptr(d), ptr(e), ptr(x), ptr(y), t.a_ptr, t.b_ptr, t.ps, t.bit, L, rows, m)


def and_finish(z, d, e, t, L, rows, m, p0):
    if _dry(z):
        return
    call("mpx_and_finish", ptr(z), ptr(d), ptr(e), t.a_ptr, t.b_ptr, t.c_ptr, t.ps, t.bit, L, rows, m, p0)


def carry_mask(dg, eg, dp, ep, G, P, t, L, rows, m, s, last):
    if _dry(dg):
        return
    call("mpx_carry_mask", ptr(dg), ptr(eg), ptr(dp), ptr(ep), ptr(G), ptr(P), t.a_ptr, t.b_ptr, t.ps,
         t.bit, L, rows, m, s, int(last))


def carry_finish(G, P, dg, eg, dp, ep, t, L, rows, m, s, last, p0):
    if _dry(G):
        return
    call("mpx_carry_finish", ptr(G), ptr(P), ptr(dg), ptr(eg), ptr(dp), ptr(ep), t.a_ptr, t.b_ptr,
         t.c_ptr, t.ps, t.bit, L, rows, m, s, int(last), p0)


def carry_fused(G, P, t, L, rows, m, s, last, p0):
    if _dry(G):
        return
    call("mpx_carry_fused", ptr(G), ptr(P), t.a_ptr, t.b_ptr, t.c_ptr, t.ps, t.bit, L, rows, m, s,
         int(last), p0)


def pubadd_init(G, P, P0, pub, x, xb_ptr, xb_ps, xb_bit, L, rows, m, p0):
    if _dry(G):
        return
    call("mpx_pubadd_init", ptr(G), ptr(P), ptr(P0), ptr(pub), ptr(x), xb_ptr, xb_ps, xb_bit, L, rows,
         m, p0)


def sum_from_carries(out, P0, G, L, rows, m):
    if _dry(out):
        return out
    call("mpx_sum_from_carries", ptr(out), ptr(P0), ptr(G), L, rows, m)
    return out


def lmo_mask(d, e, Y, t, L, rows, m, s):
    if _dry(d):
        return
    call("mpx_lmo_mask", ptr(d), ptr(e), ptr(Y), t.a_ptr, t.b_ptr, t.ps, t.bit, L, rows, m, s)


def lmo_finish(Y, d, e, t, L, rows, m, s, p0):
    if _dry(Y):
        return
    call("mpx_lmo_finish", ptr(Y), ptr(d), ptr(e), t.a_ptr, t.b_ptr, t.c_ptr, t.ps, t.bit, L, rows, m, s,
         p0)


def lmo_fused(Y, t, L, rows, m, s, p0):
    if _dry(Y):
        return
    call("mpx_lmo_fused", ptr(Y), t.a_ptr, t.b_ptr, t.c_ptr, t.ps, t.bit, L, rows, m, s, p0)


def bit2a_mask(c, b, rb_ptr, rb_ps, rb_bit, L, rows, m):
    if _dry(c):
        return c
    call("mpx_bit2a_mask", ptr(c), ptr(b), rb_ptr, rb_ps, rb_bit, L, rows, m)
    return c


def bit2a_finish(out, c, ra_ptr, ra_ps, L, rows, m, width, p0, wts=None, mode=0):
    if _dry(out):
        return out
    call("mpx_bit2a_finish", ptr(out), ptr(c), ra_ptr, ra_ps, L, rows, m, width, p0, ptr(wts), mode)
    return out


def bits_op(out, a, b, op, L, rows, m, p0=-1, imm=0):
    if _dry(out):
        return out
    call("mpx_bits_op", ptr(out), ptr(a), ptr(b), op, L, rows, m, p0, imm)
    return out


def bits_gather(out, x, src, nwords):
    if _dry(out):
        return out
    k = len(src)
    arr = (ctypes.c_int8 * 64)(*([int(s) for s in src] + [-1] * (64 - k)))
    call("mpx_bits_gather", ptr(out), ptr(x), ctypes.cast(arr, ctypes.c_void_p), k, nwords)
    return out


def bits_pack(out, x_u8, rows, m):
    if _dry(out):
        return out
    call("mpx_bits_pack", ptr(out), ptr(x_u8), rows, m)
    return out


def bits_unpack(out_u8, x, rows, m):
    if _dry(out_u8):
        return out_u8
    call("mpx_bits_unpack", ptr(out_u8), ptr(x), rows, m)
    return out_u8


def bits_flat_to_rows(out, flat_ptr, flat_bit, rows, m):
    if _dry(out):
        return out
    call("mpx_bits_flat_to_rows", ptr(out), flat_ptr, flat_bit, rows, m)
    return out


def bits_rows_to_flat(flat, rows_in, rows, m):
    if _dry(flat):
        return flat
    call("mpx_bits_rows_to_flat", ptr(flat), ptr(rows_in), rows, m)
    return flat


def im2col(out, x, L, B, C, H, W, K, stride, pad):
    if _dry(out):
        return out
    call("mpx_im2col", ptr(out), ptr(x), L, B, C, H, W, K, stride, pad)
    return out


def col2im(dx, cols, L, B, C, H, W, K, stride, pad, width):
    if _dry(dx):
        return dx
    call("mpx_col2im", ptr(dx), ptr(cols), L, B, C, H, W, K, stride, pad, width)
    return dx


# ---- GEMM -------------------------------------------------------------------

def gemm(C, A, B, batch, M, K, N, sA, sB, sC, accumulate, width, simt=False):
    """C[b] (+)= A[b] @ B[b] mod 2^w: tcgen05 limb kernel for real work, SIMT tiles otherwise."""
    if _dry(C):
        return C
    if not simt and tc_eligible(M, K, N, width):
        return gemm_tc(C, A, B, batch, M, K, N, sA, sB, sC, accumulate, width)
    call("mpx_gemm_simt" if simt else "mpx_gemm", ptr(C), A if isinstance(A, int) else ptr(A),
         B if isinstance(B, int) else ptr(B), batch, M, K, N, sA, sB, sC, int(accumulate), width)
    return C


TC_MIN_MACS = 1 << 22   # below this the SIMT tiles win (launch + split overhead)
TC_MAX_K = 16384        # exactness bound of the u32 diagonal accumulators (per CTA)


def tc_eligible(M, K, N, width) -> bool:
    return M * K * N >= TC_MIN_MACS and K >= 64 and (width == 64 or K <= TC_MAX_K or M * N >= 1 << 16)


def _rup(x, m):
    return (x + m - 1) // m * m


def kpad(kbytes: int) -> int:
    """Padded reduction length of a limb GEMM: the k-block is 32, 64 or 128
    bytes (32B / 64B / 128B swizzle), so short reductions are not padded to 128."""
    if kbytes <= 32:
        return 32
    if kbytes <= 64:
        return 64
    return _rup(kbytes, 128)


def npad_tiles(n: int) -> int:
    """Output columns the persistent kernel's N tiles cover (32-wide tile for
    outputs up to 32 wide, 64-wide tiles otherwise)."""
    return 32 if n <= 32 else _rup(n, 64)


def limb_split(out, A, rows, cols, lda, plane, pitch, coff, trans):
    if _dry(out):
        return out
    call("mpx_limb_split", ptr(out), A if isinstance(A, int) else ptr(A), rows, cols, lda, plane, pitch,
         coff, int(trans))
    return out


def ring_colsum(out, x, L, rows, cols, width):
    if _dry(out):
        return out
    call("mpx_ring_colsum", ptr(out), ptr(x), L, rows, cols, width)
    return out


def ring_pool_sum(out, x, planes, H, W, k, width, stride=None):
    if _dry(out):
        return out
    call("mpx_ring_pool_sum", ptr(out), ptr(x), planes, H, W, k, k if stride is None else stride, width)
    return out


def ring_pool_scatter(dx, d, planes, H, W, k, stride, width):
    if _dry(dx):
        return dx
    call("mpx_ring_pool_scatter", ptr(dx), ptr(d), planes, H, W, k, stride, width)
    return dx


def ring_add_rowvec(z, b, L, rows, cols, shift, width):
    if _dry(z):
        return z
    call("mpx_ring_add_rowvec", ptr(z), ptr(b), L, rows, cols, shift, width)
    return z


def beaver_gemm_batched(Z, sZ, bZ, C_ptr, sC, bC, D, E, A_ptr, sA, bA, B_ptr, sB, bB, L, batch, M, K, N, p0,
                        width):
    """``batch`` equal-shape Beaver reconstructions (one launch, all local parties)."""
    if _dry(Z):
        return Z
    call("mpx_beaver_gemm_batched", ptr(Z), sZ, bZ, C_ptr, sC, bC, ptr(D), ptr(E), A_ptr, sA, bA, B_ptr, sB, bB, L,
         batch, M, K, N, p0, width)
    return Z


def beaver_gemm_sim(Z, sZ, bZ, C_ptr, sC, bC, x_ptr, x_ps, x_sr, x_sc, x_js, A_ptr, sA, bA,
                    y_ptr, y_ps, y_sr, y_sc, y_js, B_ptr, sB, bB, L, batch, M, K, N, p0, width):
    """Sim sessions: Beaver opening + reconstruction of ``batch`` products in one launch."""
    if _dry(Z):
        return Z
    call("mpx_beaver_gemm_sim", ptr(Z), sZ, bZ, C_ptr, sC, bC, x_ptr, x_ps, x_sr, x_sc, x_js, A_ptr, sA, bA,
         y_ptr, y_ps, y_sr, y_sc, y_js, B_ptr, sB, bB, L, batch, M, K, N, p0, width)
    return Z


def beaver_tc_thin(Z, sZ, C_ptr, sC, x_ptr, x_ps, x_sr, x_sc, A_ptr, sA, y_ptr, y_ps, y_sr, y_sc, B_ptr, sB,
                   L, M, K, N, p0, width):
    """Sim sessions, K <= 32 and N <= 32: Beaver opening + reconstruction on
    tcgen05 with the limb operands built in shared memory (one launch)."""
    if _dry(Z):
        return Z
    call("mpx_beaver_tc_thin", ptr(Z), sZ, C_ptr, sC, x_ptr, x_ps, x_sr, x_sc, A_ptr, sA, y_ptr, y_ps, y_sr, y_sc,
         B_ptr, sB, L, M, K, N, p0, width)
    return Z


def beaver_tc_long(Z, sZ, C_ptr, sC, x_ptr, x_ps, x_sr, x_sc, A_ptr, sA, y_ptr, y_ps, y_sr, y_sc, B_ptr, sB,
                   L, M, K, N, p0, width, W=None):
    """Sim sessions, M <= 32 and N <= 32, long K (weight gradients of thin
    layers): split-K Beaver opening + reconstruction on tcgen05 (partials in
    the scratch W, then one launch sums them onto C)."""
    if _dry(Z):
        return Z
    need = long_tc_scratch(L, M, K, N, Z.device)
    if W is None:
        W = torch.empty(need, dtype=torch.int64, device=Z.device)
    call("mpx_beaver_tc_long", ptr(Z), sZ, C_ptr, sC, x_ptr, x_ps, x_sr, x_sc, A_ptr, sA, y_ptr, y_ps, y_sr, y_sc,
         B_ptr, sB, L, M, K, N, p0, width, ptr(W), W.numel())
    return Z


def long_tc_ok(L, M, K, N, width) -> bool:
    """Shapes mpx_beaver_tc_long takes (gemm_tc.cu long_ok)."""
    return (2 <= L <= 3 and 1 <= M <= 32 and 1 <= N <= 32 and 1 <= K < 2**31 and width == 64
            and 1024 + 81920 + 2 * L * (2 * M + 2 * N) * 34 * 8 + 64 <= 232448)


def long_tc_scratch(L, M, K, N, device) -> int:
    """Words of partial-product scratch mpx_beaver_tc_long needs."""
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    return max(sms, -(-((K + 31) // 32) // 512)) * L * M * N


def beaver_gemm(Z, sZ, C_ptr, sC, D, E, A_ptr, sA, B_ptr, sB, L, M, K, N, p0, width):
    """Z_l = C_l + D @ (B_l + [l==p0] E) + A_l @ E (one SIMT launch, all local parties)."""
    if _dry(Z):
        return Z
    call("mpx_beaver_gemm", ptr(Z), sZ, C_ptr, sC, ptr(D), ptr(E), A_ptr, sA, B_ptr, sB, L, M, K, N, p0, width)
    return Z


def beaver_limbs(A8, B8, D, E, A_ptr, a_ps, B_ptr, b_ps, L, M, K, N, Mpad, Npad, Kpad, p0):
    if _dry(A8):
        return
    call("mpx_beaver_limbs", ptr(A8), ptr(B8), ptr(D), ptr(E), A_ptr, a_ps, B_ptr, b_ps, L, M, K, N, Mpad, Npad,
         Kpad, p0)


def gemm_limbs(C, A8, B8, batch, M, N, Mpad, Npad, Kpad, ldc, sC, accumulate, width, ksplit=None,
               cin=None, s_cin=0):
    """C[z] = (C[z] if accumulate) + (Cin[z] if cin) + limb product; ``cin`` is a
    tensor or raw device address sharing C's row stride."""
    if _dry(C):
        return C
    if ksplit is None:
        ksplit = 0          # libmpx picks the split (persistent kernel: fewest waves)
    cin_ptr = None if cin is None else (cin if isinstance(cin, int) else ptr(cin))
    call("mpx_gemm_limbs", ptr(C), ptr(A8), ptr(B8), batch, M, N, Mpad, Npad, Kpad, ldc, sC,
         int(accumulate), width, int(ksplit), cin_ptr, s_cin)
    return C


def gemm_limbs_split(C, PA8, SA8, PB8, SB8, batch, M, N, Mpad, Npad, Kh, ldc, sC, width, cin, s_cin, ksplit=0,
                     zl=0, s_cin_j=0):
    """C[z] = Cin[z] + [SA[z / zl] | PA[z]] @ [PB[z] ; SB[z / zl]] on the persistent tcgen05 kernel."""
    if _dry(C):
        return C
    cin_ptr = cin if isinstance(cin, int) else ptr(cin)
    call("mpx_gemm_limbs_split", ptr(C), ptr(PA8), ptr(SA8), ptr(PB8), ptr(SB8), batch, M, N, Mpad, Npad, Kh, ldc,
         sC, width, int(ksplit), cin_ptr, s_cin, zl or batch, s_cin_j)
    return C


def mask_limbs(S8, P8, x_ptr, x_ps, x_sr, x_sc, t_ptr, t_ps, t_sr, t_sc, L, R, Kd, Rpad, Kp, p0, add_p0, width,
               jobs=1, x_js=0, t_js=0):
    """Fused sim-mode Beaver mask + limb split (shared S limbs, per-party T limbs)."""
    if _dry(S8):
        return S8
    call("mpx_mask_limbs", ptr(S8), ptr(P8), x_ptr, x_ps, x_sr, x_sc, t_ptr, t_ps, t_sr, t_sc, L, R, Kd, Rpad, Kp,
         p0, int(add_p0), width, jobs, x_js, t_js)
    return S8


def mask_limbs2(SA8, PA8, x_ptr, x_ps, x_sr, x_sc, a_ptr, a_ps, a_sr, a_sc, M, Mpad,
                SB8, PB8, y_ptr, y_ps, y_sr, y_sc, b_ptr, b_ps, b_sr, b_sc, N, Npad, L, Kd, Kp, p0, width,
                jobs=1, x_js=0, a_js=0, y_js=0, b_js=0):
    """Both operand sides of sim-mode Beaver products (mask_limbs twice) in one launch."""
    if _dry(SA8):
        return SA8
    call("mpx_mask_limbs2", ptr(SA8), ptr(PA8), x_ptr, x_ps, x_sr, x_sc, a_ptr, a_ps, a_sr, a_sc, M, Mpad,
         ptr(SB8), ptr(PB8), y_ptr, y_ps, y_sr, y_sc, b_ptr, b_ps, b_sr, b_sc, N, Npad, L, Kd, Kp, p0, width,
         jobs, x_js, a_js, y_js, b_js)
    return SA8


def gemm_tc(C, A, B, batch, M, K, N, sA, sB, sC, accumulate, width):
    """u64 GEMM on the tcgen05 limb kernel: split operands into u8 limb planes
    (scratch from the caching allocator). Width 64: one launch, split-K with
    wrapping atomics; narrower rings: K chunks of <= TC_MAX_K accumulated."""
    if _dry(C):
        return C
    dev = C.device
    Mpad, Npad = _rup(M, 128), _rup(N, 32)
    a_ptr = A if isinstance(A, int) else ptr(A)
    b_ptr = B if isinstance(B, int) else ptr(B)
    step = K if width == 64 else TC_MAX_K
    k0 = 0
    first = True
    while k0 < K:
        kc = min(step, K - k0)
        Kpad = _rup(kc, 128)
        A8 = torch.zeros((batch, 8, Mpad, Kpad), dtype=torch.uint8, device=dev)
        B8 = torch.zeros((batch, 8, Npad, Kpad), dtype=torch.uint8, device=dev)
        for z in range(batch):
            limb_split(A8[z], a_ptr + 8 * (z * sA + k0), M, kc, K, Mpad * Kpad, Kpad, 0, False)
            limb_split(B8[z], b_ptr + 8 * (z * sB + k0 * N), kc, N, N, Npad * Kpad, Kpad, 0, True)
        gemm_limbs(C, A8, B8, batch, M, N, Mpad, Npad, Kpad, N, sC, accumulate or not first, width)
        first = False
        k0 += kc
    return C


# ---- dealer -----------------------------------------------------------------

# ``key``: (k0, k1) by value, or an int64[2] device tensor (a key slot read
# at launch: the dealer's CUDA graph, preprocessing.DealerGraph)

def philox_elems(out, key, u32_off, count, width):
    if _dry(out):
        return out
    if isinstance(key, torch.Tensor):
        call("mpx_philox_elems_dk", ptr(out), ptr(key), u32_off, count, width)
    else:
        call("mpx_philox_elems", ptr(out), _u(key[0]), _u(key[1]), u32_off, count, width)
    return out


def philox_bits(out, key, u32_off, count):
    if _dry(out):
        return out
    if isinstance(key, torch.Tensor):
        call("mpx_philox_bits_dk", ptr(out), ptr(key), u32_off, count)
    else:
        call("mpx_philox_bits", ptr(out), _u(key[0]), _u(key[1]), u32_off, count)
    return out


def deal_share_arith(out, secret, key, u32_base, count, n, p_lo, L, width):
    if _dry(out):
        return out
    if isinstance(key, torch.Tensor):
        call("mpx_deal_share_arith_dk", ptr(out), out.stride(0), ptr(secret), ptr(key), u32_base, count, n, p_lo,
             L, width)
    else:
        call("mpx_deal_share_arith", ptr(out), out.stride(0), ptr(secret), _u(key[0]), _u(key[1]), u32_base,
             count, n, p_lo, L, width)
    return out


def deal_share_bits(out, secret, key, u32_base, count, n, p_lo, L):
    if _dry(out):
        return out
    if isinstance(key, torch.Tensor):
        call("mpx_deal_share_bits_dk", ptr(out), out.stride(0), ptr(secret), ptr(key), u32_base, count, n, p_lo,
             L)
    else:
        call("mpx_deal_share_bits", ptr(out), out.stride(0), ptr(secret), _u(key[0]), _u(key[1]), u32_base,
             count, n, p_lo, L)
    return out


def philox_probe(out, blocks):
    """ALU-only Philox4x64-10 throughput probe (the dealer's roofline)."""
    call("mpx_philox_probe", ptr(out), out.numel(), int(blocks))
    return out


def _key_args(key):
    """(k0, k1, dkey) for the fused dealer entry points: a key by value, or a
    device key slot (int64[2]) read at launch."""
    if isinstance(key, torch.Tensor):
        return 0, 0, ptr(key)
    return _u(key[0]), _u(key[1]), None


def deal_triple(a, b, c, key, count, n, p_lo, L, width):
    """Fused triple deal (preprocessing.py:139-145) into [L, count] share arrays."""
    if _dry(a):
        return a
    k0, k1, dk = _key_args(key)
    call("mpx_deal_triple", ptr(a), ptr(b), ptr(c), a.stride(0), k0, k1, dk, count, n, p_lo, L, width)
    return a


def deal_gen_arith(out, secret_out, key, q_secret, q_shares, count, n, p_lo, L, secret_bits, width):
    """Draw + share one secret per element (mtriple A/B, edaBit values)."""
    if _dry(out):
        return out
    k0, k1, dk = _key_args(key)
    call("mpx_deal_gen_arith", ptr(out), out.stride(0), None if secret_out is None else ptr(secret_out), k0, k1, dk,
         q_secret, q_shares, count, n, p_lo, L, secret_bits, width)
    return out


def deal_bintriple(a, b, c, key, count, n, p_lo, L):
    if _dry(a):
        return a
    k0, k1, dk = _key_args(key)
    call("mpx_deal_bintriple", ptr(a), ptr(b), ptr(c), a.stride(0), k0, k1, dk, count, n, p_lo, L)
    return a


def deal_dabit(arith, bits, key, count, n, p_lo, L, width):
    if _dry(arith):
        return arith
    k0, k1, dk = _key_args(key)
    call("mpx_deal_dabit", ptr(arith), arith.stride(0), ptr(bits), bits.stride(0), k0, k1, dk, count, n, p_lo, L,
         width)
    return arith


def deal_edabit_bits(bits, key, q_shares, count, m, width, n, p_lo, L):
    if _dry(bits):
        return bits
    k0, k1, dk = _key_args(key)
    call("mpx_deal_edabit_bits", ptr(bits), bits.stride(0), k0, k1, dk, q_shares, count, m, width, n, p_lo, L)
    return bits


def empty(shape, like: torch.Tensor):
    return torch.empty(shape, dtype=torch.int64, device=like.device)
