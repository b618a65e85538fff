/* libmpx — B200 (sm_100a) kernels for the secret-shared fixed-point engine.
 *
 * Drop-in boundary for the hot path of arXiv 2402.02320's reference package
 * `mpfix` (/root/reference/pkg/src/mpfix). The reference is pure Python +
 * numpy; its "FFI" for this path is the Python operator API
 * (protocols/__init__.py:1-30, nonlinear.py, nn.py). This C ABI is what the
 * Python host mirror (paper_2402_02320_b200/) binds through ctypes; each entry
 * point names the reference code it replaces.
 *
 * Conventions
 *  - Every function returns MPX_OK (0) or a negative MPX_ERR_* code, never
 *    allocates or frees, never synchronizes, and runs on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).
 *  - Pointers are DEVICE pointers unless the parameter name ends in `_host`.
 *  - Ring elements: uint64 words masked to `width` (w in 1..64), Z_2^w
 *    arithmetic wraps (ring.py:20-62).
 *  - Share arrays hold L local parties, party-major and contiguous:
 *    element i of local party l is at [l * n + i]. Sim mode puts all n
 *    parties on one GPU (L = n); party mode runs one process per party per
 *    GPU (L = 1).
 *  - Dealer material arrays carry their own party stride `*_ps` (elements or
 *    words) and the host passes pointers already advanced to the store cursor
 *    (preprocessing.py:281-291). Bit material is a flat packed bit stream per
 *    party (bit t = item t) and is addressed by absolute bit offset `*_bit`.
 *  - Binary shares are row-packed: one uint64 word per row, low `m` bits are
 *    the row's trailing bit axis, LSB first (ring.py:110-114).
 *  - `p0` = local slot of party 0, or -1 when party 0 is not local: public
 *    constants land on party 0 only (sharing.py:99-121).
 */
#ifndef MPX_H_
#define MPX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPX_OK 0
#define MPX_ERR_ARG (-1)
#define MPX_ERR_CUDA (-2)
#define MPX_ERR_UNSUPPORTED (-3)

/* bit-op codes for mpx_bits_op */
#define MPX_BITS_XOR 0      /* out = a ^ b                                   */
#define MPX_BITS_AND 1      /* out = a & b                                   */
#define MPX_BITS_AND_PUB 2  /* out = a & pub[row]        (sharing.py:84-86)  */
#define MPX_BITS_XOR_PUB 3  /* out = a ^ [p0] pub[row]   (sharing.py:99-103) */
#define MPX_BITS_XOR_SHR1 4 /* out = a ^ (a >> 1)        (derived.py:148)    */
#define MPX_BITS_PARITY 5   /* out = popcount(a & mask(m)) & 1 (nonlinear.py:243) */
#define MPX_BITS_SIGNFOLD 6 /* out = (a & mask(m)) ^ (bit m of a ? mask(m):0) (nonlinear.py:162) */
#define MPX_BITS_SHL_OR 7   /* out = (a & mask(imm)) | (b << imm)  (bit-axis concat) */
#define MPX_BITS_BCAST_PUB 8 /* out = a ^ [p0] pub[0]  (public constant pattern) */

/* Library identity / diagnostics. */
const char* mpx_version(void);
int mpx_last_cuda_error(void);
const char* mpx_cuda_error_string(int code);
int mpx_device_sm_count(int device);

/* ---- local ring arithmetic (ring.py:44-62, sharing.py:37-56,99-121) ---- */
/* out[l][i] = ka*a[l][i] + kb*b[l][i] + [l==p0](c0 + cv[i % cv_len])  mod 2^w.
 * b and cv may be NULL. Covers add/sub/neg/mul_public/add_public/add_const/
 * scale_fixed (derived.py:73-83) and narrow/cast_down (nn.py:68-74). */
int mpx_ring_lin(uint64_t* out, const uint64_t* a, uint64_t ka, const uint64_t* b, uint64_t kb,
                 uint64_t c0, const uint64_t* cv, int64_t cv_len, int L, int64_t n, int width, int p0,
                 void* stream);
/* out[i] = a[i] * b[i] mod 2^w (public elementwise product; dealer c = a*b,
 * preprocessing.py:141). */
int mpx_ring_mul(uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, int width, void* stream);
/* out[l][r] = sum_j wts[j] * x[l][r][j] mod 2^w; wts NULL = all ones.
 * Row sums (nn.py:134), compose weights (basic.py:193-195), one-hot
 * contractions (nonlinear.py:117-122, 252-256). */
int mpx_ring_rowdot(uint64_t* out, const uint64_t* x, const uint64_t* wts, int L, int64_t rows,
                    int64_t cols, int width, void* stream);
/* out[l][c] = sum_r x[l][r][c] mod 2^width, x: [L][rows][cols] (bias gradients). */
int mpx_ring_colsum(uint64_t* out, const uint64_t* x, int L, int64_t rows, int64_t cols, int width,
                    void* stream);
/* k x k window sums, stride st, over [planes][H][W] -> [planes][OH][OW] with
 * OH = (H - k) / st + 1 (average pooling before its 1/k^2 scaling). */
int mpx_ring_pool_sum(uint64_t* out, const uint64_t* x, int64_t planes, int64_t H, int64_t W, int64_t k,
                      int64_t stride, int width, void* stream);
/* Adjoint: dx[p][h][w] = sum of d[p][oi][oj] over the windows covering (h, w). */
int mpx_ring_pool_scatter(uint64_t* dx, const uint64_t* d, int64_t planes, int64_t H, int64_t W, int64_t k,
                          int64_t stride, int width, void* stream);
/* z[l][r][c] = z[l][r][c] + (b[l][c] << shift) mod 2^width, in place (bias rows). */
int mpx_ring_add_rowvec(uint64_t* z, const uint64_t* b, int L, int64_t rows, int64_t cols, int shift,
                        int width, void* stream);

/* ---- fixed-point codec (ring.py:76-89) ---- */
int mpx_encode(uint64_t* out, const double* in, int64_t n, int width, int frac, void* stream);
int mpx_decode(double* out, const uint64_t* in, int64_t n, int width, int frac, void* stream);
/* ring.to_signed (ring.py:65-73): centered int64 representative of Z_2^w words. */
int mpx_to_signed(int64_t* out, const uint64_t* in, int64_t n, int width, void* stream);

/* ---- openings: local-party reduction of one round (session.py:71-115) ----
 * Sim mode: the reduction over all L parties IS the opening. Party mode: the
 * partial is all-reduced (sum) / all-gathered (xor) over NCCL by the host. */
int mpx_open_sum(uint64_t* out, const uint64_t* x, int L, int64_t n, int width, void* stream);
int mpx_open_xor(uint64_t* out, const uint64_t* x, int L, int64_t n, void* stream);
/* out[i] = sum_l (x[l][i] - a[l][i]) mod 2^w: the masked opening of Beaver
 * mul/matmul (basic.py:36, :66) and decompose (basic.py:211). */
int mpx_mask_sub(uint64_t* out, const uint64_t* x, const uint64_t* a, int64_t a_ps, int L, int64_t n,
                 int width, void* stream);
/* Batched, strided masks (every equal-shape product of a batch_matmul round):
 * out[b][j] = sum_l (x_l[b][j] - a_l[b][j]); x at party / batch strides
 * x_ps / x_bs, a at a_ps / a_bs; out contiguous [batch][n]. */
int mpx_mask_sub_bs(uint64_t* out, const uint64_t* x, int64_t x_ps, int64_t x_bs, const uint64_t* a,
                    int64_t a_ps, int64_t a_bs, int L, int64_t batch, int64_t n, int width, void* stream);
/* Transposed operands read in place: out[b][r][c] = sum_l (x_l[b][c][r] - a_l[b][r][c])
 * (Beaver masks of X^T, W^T, K^T). */
int mpx_mask_sub_t(uint64_t* out, const uint64_t* x, int64_t x_ps, int64_t x_bs, const uint64_t* a,
                   int64_t a_ps, int64_t a_bs, int L, int64_t batch, int64_t rows, int64_t cols, int width,
                   void* stream);

/* ---- Beaver multiplication (basic.py:27-42) ----
 * z_l = c_l + d*b_l + e*a_l + [l==p0] d*e. */
int mpx_mul_finish(uint64_t* z, const uint64_t* d, const uint64_t* e, const uint64_t* a,
                   const uint64_t* b, const uint64_t* c, int64_t t_ps, int L, int64_t n, int width,
                   int p0, void* stream);
/* Fused sim-mode round (L parties on this GPU, no peer): mask, open and
 * finish in one pass. */
int mpx_mul_fused(uint64_t* z, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                  const uint64_t* b, const uint64_t* c, int64_t t_ps, int L, int64_t n, int width,
                  int p0, void* stream);

/* ---- probabilistic truncation (derived.py:20-70) ----
 * mask: out[i] = sum_l (x + r_lo + 2^f r_hi + [l==p0] bias)   (r_hi may be NULL)
 * finish: z_l = -r_hi_l + [l==p0]((c >> f) - unbias)            mod 2^w */
int mpx_trunc_mask(uint64_t* out, const uint64_t* x, const uint64_t* r_lo, int64_t lo_ps,
                   const uint64_t* r_hi, int64_t hi_ps, int L, int64_t n, int width, int f,
                   uint64_t bias, int p0, void* stream);
int mpx_trunc_finish(uint64_t* z, const uint64_t* c, const uint64_t* r_hi, int64_t hi_ps, int L,
                     int64_t n, int width, int f, uint64_t unbias, int p0, void* stream);
int mpx_trunc_fused(uint64_t* z, const uint64_t* x, const uint64_t* r_lo, int64_t lo_ps,
                    const uint64_t* r_hi, int64_t hi_ps, int L, int64_t n, int width, int f,
                    uint64_t bias, uint64_t unbias, int p0, void* stream);
/* Up to 16 independent sim-mode truncations in one launch; each job is
 * z = trunc(x) or, with a base, z = base - trunc(x) (SGD updates). jobs_host
 * points to a host TruncJobs {TruncJob j[16]; int64_t start[17]; int n, pad}
 * with TruncJob {z, base, x, r_lo, r_hi, lo_ps, hi_ps, n, bias, unbias, f, pad}. */
int mpx_trunc_sub_multi(const void* jobs_host, int L, int width, int p0, void* stream);
/* Sim-mode truncation of x[l][b*S+s][c] + (brow[l][c] << bshift) (a layer's
 * product plus its lifted bias row, brow may be null), material in that row
 * order; nchw = 1 stores z[l][b][c][s] (conv output), 0 stores rows. L <= 4. */
int mpx_trunc_rows_bias(uint64_t* z, const uint64_t* x, const uint64_t* brow, int bshift, const uint64_t* r_lo,
                        int64_t lo_ps, const uint64_t* r_hi, int64_t hi_ps, int L, int64_t B, int64_t S,
                        int64_t C, int nchw, int width, int f, uint64_t bias, uint64_t unbias, int p0,
                        void* stream);
/* Sim-mode truncation of an NCHW tensor x[l][b][c][hs][ws], each value
 * broadcast to its k x k window in conv row order z[l][(b*H+h)*W+w][c]
 * (average-pool backward feeding a conv backward). L <= 4. */
int mpx_trunc_expand_rows(uint64_t* z, const uint64_t* x, const uint64_t* r_lo, int64_t lo_ps,
                          const uint64_t* r_hi, int64_t hi_ps, int L, int64_t B, int64_t C, int64_t Hs,
                          int64_t Ws, int64_t k, int width, int f, uint64_t bias, uint64_t unbias, int p0,
                          void* stream);

/* ---- binary Beaver AND on row-packed bits (basic.py:82-95) ----
 * triple for (row r, bit j) = bit (t_bit + r*m + j) of the bintriple stream. */
int mpx_and_mask(uint64_t* d, uint64_t* e, const uint64_t* x, const uint64_t* y, const uint64_t* ta,
                 const uint64_t* tb, int64_t t_ps, int64_t t_bit, int L, int64_t rows, int m,
                 void* stream);
int mpx_and_finish(uint64_t* z, const uint64_t* d, const uint64_t* e, const uint64_t* ta,
                   const uint64_t* tb, const uint64_t* tc, int64_t t_ps, int64_t t_bit, int L,
                   int64_t rows, int m, int p0, void* stream);

/* ---- Kogge-Stone carry level (basic.py:98-129) at shift s over m bits ----
 * Non-final level: one AND call on [p_hi|p_hi] & [g_lo|p_lo] (row width
 * 2(m-s)); final level: p_hi & g_lo (row width m-s). G, P updated in place.
 * dg/eg/dp/ep: opened masked words (dp/ep unused on the final level). */
int mpx_carry_mask(uint64_t* dg, uint64_t* eg, uint64_t* dp, uint64_t* ep, const uint64_t* G,
                   const uint64_t* P, const uint64_t* ta, const uint64_t* tb, int64_t t_ps,
                   int64_t t_bit, int L, int64_t rows, int m, int s, int last, void* stream);
int mpx_carry_finish(uint64_t* G, uint64_t* P, const uint64_t* dg, const uint64_t* eg,
                     const uint64_t* dp, const uint64_t* ep, const uint64_t* ta, const uint64_t* tb,
                     const uint64_t* tc, int64_t t_ps, int64_t t_bit, int L, int64_t rows, int m,
                     int s, int last, int p0, void* stream);
int mpx_carry_fused(uint64_t* G, uint64_t* P, const uint64_t* ta, const uint64_t* tb,
                    const uint64_t* tc, int64_t t_ps, int64_t t_bit, int L, int64_t rows, int m,
                    int s, int last, int p0, void* stream);
/* Public-operand adder set-up (basic.py:139-152): G = x & pub, P = P0 = x ^ [p0] pub.
 * x comes from `x` (row words, L x rows) or, when x == NULL, from the edaBit
 * bit stream xb (bit xb_bit + r*m + j) as in decompose (basic.py:199-214). */
int mpx_pubadd_init(uint64_t* G, uint64_t* P, uint64_t* P0, const uint64_t* pub, const uint64_t* x,
                    const uint64_t* xb, int64_t xb_ps, int64_t xb_bit, int L, int64_t rows, int m,
                    int p0, void* stream);
/* sum = P0 ^ (carries << 1)  (basic.py:132-136) */
int mpx_sum_from_carries(uint64_t* out, const uint64_t* P0, const uint64_t* G, int L, int64_t rows,
                         int m, void* stream);

/* ---- leftmost-one suffix-OR level (derived.py:131-149) ----
 * lo = Y[:m-s], hi = Y[s:]; Y[:m-s] = lo ^ hi ^ AND(lo, hi). */
int mpx_lmo_mask(uint64_t* d, uint64_t* e, const uint64_t* Y, const uint64_t* ta, const uint64_t* tb,
                 int64_t t_ps, int64_t t_bit, int L, int64_t rows, int m, int s, void* stream);
int mpx_lmo_finish(uint64_t* Y, const uint64_t* d, const uint64_t* e, const uint64_t* ta,
                   const uint64_t* tb, const uint64_t* tc, int64_t t_ps, int64_t t_bit, int L,
                   int64_t rows, int m, int s, int p0, void* stream);
int mpx_lmo_fused(uint64_t* Y, const uint64_t* ta, const uint64_t* tb, const uint64_t* tc,
                  int64_t t_ps, int64_t t_bit, int L, int64_t rows, int m, int s, int p0,
                  void* stream);

/* ---- daBit conversion (basic.py:164-196) ----
 * mask: c[r] = xor_l (b_l[r] ^ rbits_l(r)) ; daBit (r, j) = bit rb_bit + r*m + j.
 * finish: z = r_arith*(1-2c) + [p0] c ; mode 0 writes z as (L, rows, m),
 * mode 1 writes sum_j wts[j]*z (L, rows) (compose). */
int mpx_bit2a_mask(uint64_t* c, const uint64_t* b, const uint64_t* rbits, int64_t rb_ps,
                   int64_t rb_bit, int L, int64_t rows, int m, void* stream);
int mpx_bit2a_finish(uint64_t* out, const uint64_t* c, const uint64_t* rarith, int64_t ra_ps, int L,
                     int64_t rows, int m, int width, int p0, const uint64_t* wts, int mode,
                     void* stream);

/* ---- local bit manipulation on row-packed words ---- */
int mpx_bits_op(uint64_t* out, const uint64_t* a, const uint64_t* b, int op, int L, int64_t rows,
                int m, int p0, int imm, void* stream);
/* out[i] bit t = in[i] bit src_host[t] (src < 0 -> 0), t < k. Slicing,
 * reversal and bit selection of the trailing axis (nonlinear.py:170,199,344). */
int mpx_bits_gather(uint64_t* out, const uint64_t* in, const int8_t* src_host, int k, int64_t nwords,
                    void* stream);
/* uint8-per-bit (rows, m) <-> row-packed words (BShare layout conversion). */
int mpx_bits_pack(uint64_t* out, const uint8_t* in, int64_t rows, int m, void* stream);
int mpx_bits_unpack(uint8_t* out, const uint64_t* in, int64_t rows, int m, void* stream);
/* Flat bit stream (bit t) -> row words (m bits per row) and back. */
int mpx_bits_flat_to_rows(uint64_t* out, const uint64_t* flat, int64_t flat_bit, int64_t rows, int m,
                          void* stream);
int mpx_bits_rows_to_flat(uint64_t* flat, const uint64_t* rows_in, int64_t rows, int m, void* stream);

/* ---- convolution layout on shares (CNN layers) ----
 * x: [L][B][C][H][W] -> cols: [L][B*OH*OW][C*K*K] (zero padding), and the
 * adjoint scatter-add col2im (mod 2^w). Local: no communication. */
int mpx_im2col(uint64_t* out, const uint64_t* x, int L, int64_t B, int C, int H, int W, int K, int stride,
               int pad, void* stream);
int mpx_col2im(uint64_t* dx, const uint64_t* cols, int L, int64_t B, int C, int H, int W, int K, int stride,
               int pad, int width, void* stream);

/* ---- Z_2^64 GEMM (ring.py:60-62; basic.py:72-75; nn.py:193) ----
 * C[b] (+)= A[b] @ B[b] mod 2^w, row-major, A: MxK, B: KxN, C: MxN,
 * batch strides sA/sB/sC in elements (0 broadcasts). */
int mpx_gemm(uint64_t* C, const uint64_t* A, const uint64_t* B, int64_t batch, int64_t M, int64_t K,
             int64_t N, int64_t sA, int64_t sB, int64_t sC, int accumulate, int width, void* stream);
/* Same contract, forced onto the exact 64-bit SIMT tiles (reference shape). */
int mpx_gemm_simt(uint64_t* C, const uint64_t* A, const uint64_t* B, int64_t batch, int64_t M,
                  int64_t K, int64_t N, int64_t sA, int64_t sB, int64_t sC, int accumulate, int width,
                  void* stream);

/* ---- tcgen05 int8-limb Z_2^64 GEMM (gemm_tc.cu) ----
 * Limb split of a row-major u64 matrix into 8 u8 planes (plane stride
 * `plane`, padded K `pitch` bytes, `coff` must be 0): trans = 0 writes row r,
 * K byte c; trans = 1 writes row c, K byte r (K-major B). Planes are K-block
 * tiled: byte k of row r at ((k / tw) * Rpad + r) * tw + k % tw with
 * tw = min(128, pitch), Rpad = plane / pitch, so each TMA box of the GEMM is
 * one contiguous run of HBM. */
int mpx_limb_split(uint8_t* out, const uint64_t* A, int64_t rows, int64_t cols, int64_t lda,
                   int64_t plane, int64_t pitch, int64_t coff, int trans, void* stream);
/* Beaver matmul operands for all L parties in two launches: A8[l] = limbs
 * of [D | A_l] (M x 2K), B8[l] = limbs of [B_l + [l==p0] E ; E]^T (N x 2K);
 * planes K-block tiled like mpx_limb_split's; padding rows and columns are
 * written as zeros. */
int mpx_beaver_limbs(uint8_t* A8, uint8_t* B8, const uint64_t* D, const uint64_t* E, const uint64_t* A,
                     int64_t a_ps, const uint64_t* B, int64_t b_ps, int L, int64_t M, int64_t K, int64_t N,
                     int64_t Mpad, int64_t Npad, int64_t Kpad, int p0, void* stream);
/* C[z] (+)= sum_{i+j<=7} 2^(8(i+j)) A8[z][i] @ B8[z][j]^T mod 2^w on tcgen05
 * kind::i8 with per-diagonal TMEM accumulators, TMA-fed (128B swizzle).
 * A8: [batch][8][Mpad][Kpad], B8: [batch][8][Npad][Kpad] u8, zero padded;
 * Mpad % 128 == 0, Npad % 32 == 0, Kpad % 128 == 0. Persistent (one CTA per
 * SM) over 128 x 64 tiles x split-K slices (each <= 16384 of K, the
 * exactness bound) that add their u64 partials with wrapping atomics (width
 * 64 only); ksplit 0 = automatic (fewest waves), >= 1 forced. */
int mpx_gemm_limbs(uint64_t* C, const uint8_t* A8, const uint8_t* B8, int64_t batch, int64_t M,
                   int64_t N, int64_t Mpad, int64_t Npad, int64_t Kpad, int64_t ldc, int64_t sC,
                   int accumulate, int width, int ksplit, const uint64_t* Cin, int64_t sCin,
                   void* stream);

/* Split-operand variant (sim sessions, operands from mpx_mask_limbs):
 * C[z] = Cin[z] + [SA | PA[z]] @ [PB[z] ; SB] mod 2^w, SA / SB shared
 * [8][rows][Kh] limb planes, PA / PB per party [batch][8][rows][Kh]; i.e.
 * basic.py:72-75 with D, E limbs stored once for all parties. Kh % 128 == 0,
 * ksplit 0 = automatic. Several equal-shape products in one launch: batch =
 * jobs x zl parties, unit z uses shared plane set z / zl and addend
 * Cin + (z % zl) * sCin + (z / zl) * sCin_j. */
int mpx_gemm_limbs_split(uint64_t* C, const uint8_t* PA8, const uint8_t* SA8, const uint8_t* PB8,
                         const uint8_t* SB8, int64_t batch, int64_t M, int64_t N, int64_t Mpad, int64_t Npad,
                         int64_t Kh, int64_t ldc, int64_t sC, int width, int ksplit, const uint64_t* Cin,
                         int64_t sCin, int zl, int64_t sCin_j, void* stream);
/* Fused Beaver mask + limb split for an all-parties-local session (the
 * opening of basic.py:66-70 is a local reduction): S8 = limbs of
 * S = sum_l (X_l - T_l) mod 2^w, P8[l] = limbs of T_l (+ S at party p0 when
 * add_p0). X_l, T_l: logical R x K at (row, col) strides (transposed views
 * read in place), party strides x_ps / t_ps; planes K-major [Rpad][Kp],
 * zero padded (Rpad % 32 == 0, Kp % 32 == 0). `jobs` equal-shape operand
 * pairs at element strides x_js / t_js in one launch; job j writes plane
 * sets S8 + j * 8 * Rpad * Kp and P8 + j * L * 8 * Rpad * Kp. */
int mpx_mask_limbs(uint8_t* S8, uint8_t* P8, const uint64_t* X, int64_t x_ps, int64_t x_sr, int64_t x_sc,
                   const uint64_t* T, int64_t t_ps, int64_t t_sr, int64_t t_sc, int L, int64_t R, int64_t K,
                   int64_t Rpad, int64_t Kp, int p0, int add_p0, int width, int jobs, int64_t x_js,
                   int64_t t_js, void* stream);

/* Both sides of a sim-mode Beaver product in ONE launch (basic.py:66-70):
 * side A = mpx_mask_limbs(SA8, PA8, X, A; R = M, Rpad = Mpad, add_p0 = 0),
 * side B = mpx_mask_limbs(SB8, PB8, Y^T, B^T; R = N, Rpad = Npad,
 * add_p0 = 1), same L, K, Kp, p0, width and job count (job strides
 * x_js / a_js / y_js / b_js). */
int mpx_mask_limbs2(uint8_t* SA8, uint8_t* PA8, const uint64_t* X, int64_t x_ps, int64_t x_sr, int64_t x_sc,
                    const uint64_t* A, int64_t a_ps, int64_t a_sr, int64_t a_sc, int64_t M, int64_t Mpad,
                    uint8_t* SB8, uint8_t* PB8, const uint64_t* Y, int64_t y_ps, int64_t y_sr, int64_t y_sc,
                    const uint64_t* B, int64_t b_ps, int64_t b_sr, int64_t b_sc, int64_t N, int64_t Npad, int L,
                    int64_t K, int64_t Kp, int p0, int width, int jobs, int64_t x_js, int64_t a_js, int64_t y_js,
                    int64_t b_js, void* stream);

/* Sim sessions (all L local parties, 2 <= L <= 4): the Beaver opening and
 * reconstruction of `batch` equal-shape products in one launch
 * (basic.py:66-75): D = sum_l (X_l - A_l), E = sum_l (Y_l - B_l) formed in
 * shared memory, Z_l = C_l + D @ (B_l + [l==p0] E) + A_l @ E mod 2^width.
 * X / Y: logical M x K / K x N views at (party, row, col, job) element
 * strides; A_l (M x K), B_l (K x N), C_l, Z_l (M x N) row-major at party
 * strides sA / sB / sC / sZ and job strides bA / bB / bC / bZ. */
int mpx_beaver_gemm_sim(uint64_t* Z, int64_t sZ, int64_t bZ, const uint64_t* C, int64_t sC, int64_t bC,
                        const uint64_t* X, int64_t x_ps, int64_t x_sr, int64_t x_sc, int64_t x_js,
                        const uint64_t* A, int64_t sA, int64_t bA, const uint64_t* Y, int64_t y_ps, int64_t y_sr,
                        int64_t y_sc, int64_t y_js, const uint64_t* B, int64_t sB, int64_t bB, int L,
                        int64_t batch, int64_t M, int64_t K, int64_t N, int p0, int width, void* stream);

/* Beaver matrix-product reconstruction in one launch (basic.py:72-75):
 * Z_l = C_l + D @ (B_l + [l==p0] E) + A_l @ E mod 2^width for the L local
 * parties (batch strides sZ, sC, sA, sB). Z, C: M x N; D, A: M x K; E, B:
 * K x N, all row-major. SIMT u64 tiles sized to the output (thin layers),
 * split-K with wrapping atomics for tiny outputs (width 64). */
int mpx_beaver_gemm(uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* D,
                    const uint64_t* E, const uint64_t* A, int64_t sA, const uint64_t* B, int64_t sB,
                    int L, int64_t M, int64_t K, int64_t N, int p0, int width, void* stream);
/* `batch` independent equal-shape reconstructions in one launch; product b
 * uses Z + b*bZ, C + b*bC, D + b*M*K, E + b*K*N, A + b*bA, B + b*bB. */
int mpx_beaver_gemm_batched(uint64_t* Z, int64_t sZ, int64_t bZ, const uint64_t* C, int64_t sC, int64_t bC,
                            const uint64_t* D, const uint64_t* E, const uint64_t* A, int64_t sA, int64_t bA,
                            const uint64_t* B, int64_t sB, int64_t bB, int L, int64_t batch, int64_t M,
                            int64_t K, int64_t N, int p0, int width, void* stream);

/* ---- sim-mode whole-op fused kernels (fused_ops.cu) ----
 * All L parties on this GPU: the whole Reciprocal / Exp / Log protocol
 * (nonlinear.py:146-267) runs in one kernel, one thread per element, shares
 * in registers. `tape_host` points to a host `Tape` (one MatRef per dealer
 * take, in protocol order) and `params_host` to `FusedParams`; layouts are
 * reported by mpx_fused_abi_sizes. */
int mpx_reciprocal_fused(uint64_t* y, const uint64_t* x, int64_t n, const void* tape_host,
                         const void* params_host, void* stream);
int mpx_exp_fused(uint64_t* y, const uint64_t* x, int64_t n, const void* tape_host,
                  const void* params_host, void* stream);
int mpx_log_fused(uint64_t* y, const uint64_t* x, int64_t n, const void* tape_host,
                  const void* params_host, void* stream);
/* attention_exp (nonlinear.py:315-356): 32-bit ring input, 64-bit ring output. */
int mpx_attexp_fused(uint64_t* y, const uint64_t* x, int64_t n, const void* tape_host,
                     const void* params_host, void* stream);
/* ReLU (nn.py:92-97) in one kernel: y = bit2a(gt(x, 0)) * x; when s_out is
 * non-null the converted sign is stored too (training backward). */
int mpx_relu_fused(uint64_t* y, uint64_t* s_out, const uint64_t* x, int64_t n, const void* tape_host,
                   const void* params_host, void* stream);
/* One max tournament level (derived.py:152-170): win = v + bit2a(gt(u, v)) * (u - v). */
int mpx_maxlevel_fused(uint64_t* win, const uint64_t* u, const uint64_t* v, int64_t n,
                       const void* tape_host, const void* params_host, void* stream);
/* A whole max_vec tournament (derived.py:152-170) of `rows` rows of width d0
 * (<= 512) in one launch: one CTA per row, level by level in shared memory;
 * `levels_host` holds each level's first tape index (the per-level tapes
 * concatenated, so material order equals the per-level kernels'). */
int mpx_maxtour_fused(uint64_t* y, const uint64_t* x, int64_t rows, int d0, const void* tape_host,
                      const void* levels_host, const void* params_host, void* stream);
int mpx_fused_tour_size(int64_t* levels);
/* softmax_parts (nn.py:115-136) in one launch, one CTA per row (d0 <= 256):
 * [rescale by log2 e], narrow to 32 bits, max tournament, x - max - 1 ulp,
 * attention_exp, row sum, reciprocal. `segs_host` (SoftmaxSegs) holds each
 * stage's first tape index; the three FusedParams are the tournament's,
 * attention-exp's and reciprocal's. Outputs e (like x) and r (one per row). */
int mpx_softmax_fused(uint64_t* e_out, uint64_t* r_out, const uint64_t* x, int64_t rows, int d0,
                      const void* tape_host, const void* segs_host, const void* pm_host, const void* pe_host,
                      const void* pr_host, void* stream);
int mpx_fused_softmax_size(int64_t* segs);
int mpx_fused_abi_sizes(int64_t* matref, int64_t* tape, int64_t* params, int64_t* tape_max);

/* ---- trusted dealer (preprocessing.py:121-174; ring.py:124-134) ----
 * Philox4x64-10 keyed (k0, k1) exactly as numpy; the byte stream is read as
 * u32 words from u32 index `u32_off` (Generator.bytes semantics). */
int mpx_philox_elems(uint64_t* out, uint64_t k0, uint64_t k1, int64_t u32_off, int64_t count,
                     int width, void* stream);
int mpx_philox_bits(uint64_t* out_words, uint64_t k0, uint64_t k1, int64_t u32_off, int64_t count,
                    void* stream);
/* Additive shares of `secret` (count elems) for global parties p_lo..p_lo+L-1:
 * party p < n-1 gets draw p (u32 offset u32_base + p*2*count), the last party
 * gets secret - sum(draws) (sharing.py:124-133). */
int mpx_deal_share_arith(uint64_t* out, int64_t out_ps, const uint64_t* secret, uint64_t k0,
                         uint64_t k1, int64_t u32_base, int64_t count, int n, int p_lo, int L,
                         int width, void* stream);
/* XOR shares of a packed bit stream `secret_words` (count bits); draw k at
 * u32 offset u32_base + k*ceil(count/4) (sharing.py:144-152). */
int mpx_deal_share_bits(uint64_t* out, int64_t out_ps, const uint64_t* secret_words, uint64_t k0,
                        uint64_t k1, int64_t u32_base, int64_t count, int n, int p_lo, int L,
                        void* stream);
/* The same four draws with the Philox key read from a device slot
 * dkey[0..1] at launch: a CUDA graph of a whole re-deal replays with fresh
 * keys written into the slots (preprocessing.py:121-125 keys per seed). */
int mpx_philox_elems_dk(uint64_t* out, const uint64_t* dkey, int64_t u32_off, int64_t count, int width,
                        void* stream);
int mpx_philox_bits_dk(uint64_t* out_words, const uint64_t* dkey, int64_t u32_off, int64_t count,
                       void* stream);
int mpx_deal_share_arith_dk(uint64_t* out, int64_t out_ps, const uint64_t* secret, const uint64_t* dkey,
                            int64_t u32_base, int64_t count, int n, int p_lo, int L, int width, void* stream);
int mpx_deal_share_bits_dk(uint64_t* out, int64_t out_ps, const uint64_t* secret_words, const uint64_t* dkey,
                           int64_t u32_base, int64_t count, int n, int p_lo, int L, void* stream);

/* Thin sim-mode Beaver product on tcgen05 (basic.py:66-75), operand limbs
 * built in shared memory: Z_l = C_l + [D | A_l] @ [B_l + [l==p0] E ; E] with
 * D = sum_l X_l - A_l, E = sum_l Y_l - B_l, for K <= 32, N <= 32, L = 2..3
 * local parties (LeNet conv1 forward). Z, C [L][M][N], A [L][M][K],
 * B [L][K][N] at party strides; X (M x K), Y (K x N) at (party, row, col)
 * strides. */
int mpx_beaver_tc_thin(uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* X,
                       int64_t x_ps, int64_t x_sr, int64_t x_sc, const uint64_t* A, int64_t sA,
                       const uint64_t* Y, int64_t y_ps, int64_t y_sr, int64_t y_sc, const uint64_t* B,
                       int64_t sB, int L, int64_t M, int64_t K, int64_t N, int p0, int width, void* stream);

/* Long-K small sim-mode Beaver product on tcgen05 (basic.py:66-75): same
 * operands and result as mpx_beaver_tc_thin, for M <= 32, N <= 32, any K,
 * L = 2..3 local parties, width 64 (LeNet conv1 weight gradient, K = 73728).
 * Split-K over the SMs: every CTA writes its partial product into the scratch
 * W (at least max(SMs, ceil(K / 16384)) * L * M * N words) and a second
 * launch sums the partials onto C. Shared-memory budget:
 * 1024 + 81920 + 16 L (2M + 2N) * 34 + 64 <= 232448. */
int mpx_beaver_tc_long(uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* X,
                       int64_t x_ps, int64_t x_sr, int64_t x_sc, const uint64_t* A, int64_t sA,
                       const uint64_t* Y, int64_t y_ps, int64_t y_sr, int64_t y_sc, const uint64_t* B,
                       int64_t sB, int L, int64_t M, int64_t K, int64_t N, int p0, int width, uint64_t* W,
                       int64_t w_words, void* stream);

/* Philox4x64-10 ALU ceiling probe: `blocks` counter blocks generated and
 * XOR-folded into out[grid*256] (out_words >= 148*8*256), no other memory
 * traffic: the dealer's roofline denominator, measured in-run. */
int mpx_philox_probe(uint64_t* out, int64_t out_words, int64_t blocks, void* stream);

/* ---- fused per-kind dealer: ONE launch per material key ----
 * Each thread draws its group's secrets straight from the key's stream (draw
 * order SURVEY App. A4 / preprocessing.py:139-171), derives c = a*b or
 * c = a & b in registers and writes only the local parties' shares
 * (p_lo..p_lo+L-1; party stride `ps` elements or words). `dkey` (nullable)
 * overrides (k0, k1) with a device key slot read at launch (CUDA-graph
 * re-deals). Replaces the draw -> store -> share kernel chains above. */
/* triple (preprocessing.py:139-145): out a, b, c [L][count] */
int mpx_deal_triple(uint64_t* a, uint64_t* b, uint64_t* c, int64_t ps, uint64_t k0, uint64_t k1,
                    const uint64_t* dkey, int64_t count, int n, int p_lo, int L, int width, void* stream);
/* one drawn secret per element at u32 offset q_secret, masked to
 * min(width, secret_bits) bits, optionally stored to secret_out (count
 * elems), shared with draws at q_shares + p*2*count: mtriple A / B
 * (preprocessing.py:146-152) and edaBit values + arithmetic shares (:165-170). */
int mpx_deal_gen_arith(uint64_t* out, int64_t ps, uint64_t* secret_out, uint64_t k0, uint64_t k1,
                       const uint64_t* dkey, int64_t q_secret, int64_t q_shares, int64_t count, int n,
                       int p_lo, int L, int secret_bits, int width, void* stream);
/* bintriple (preprocessing.py:153-159): packed bit streams a, b, c [L][words] */
int mpx_deal_bintriple(uint64_t* a, uint64_t* b, uint64_t* c, int64_t ps, uint64_t k0, uint64_t k1,
                       const uint64_t* dkey, int64_t count, int n, int p_lo, int L, void* stream);
/* daBit (preprocessing.py:160-164): arithmetic shares [L][count], bit shares [L][words] */
int mpx_deal_dabit(uint64_t* arith, int64_t arith_ps, uint64_t* bit_words, int64_t bit_ps, uint64_t k0,
                   uint64_t k1, const uint64_t* dkey, int64_t count, int n, int p_lo, int L, int width,
                   void* stream);
/* edaBit bit shares (preprocessing.py:165-170): the m low bits of each value
 * (value draw at u32 offset 0) as a packed stream, shared with draws of
 * count*m bytes at q_shares. */
int mpx_deal_edabit_bits(uint64_t* bit_words, int64_t ps, uint64_t k0, uint64_t k1, const uint64_t* dkey,
                         int64_t q_shares, int64_t count, int m, int width, int n, int p_lo, int L,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPX_H_ */
