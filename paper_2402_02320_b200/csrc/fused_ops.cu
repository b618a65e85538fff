// Whole-op fused kernels for the all-parties-on-one-GPU deployment (sim mode).
//
// With every party's shares on this GPU an opening needs no communication, so
// the 23-37 rounds of Exp / Log / Reciprocal can run inside ONE kernel: each
// thread owns one element and keeps all L parties' shares in registers from
// the input to the output, reading each item of its dealer material exactly
// once. The protocol is the reference's, step for step (nonlinear.py:146-267,
// basic.py:27-214, derived.py:20-149); the host records the exact sequence of
// material takes (a "tape": one MatRef per take, pointers already advanced to
// the store cursor) by running the Python protocol as a dry pass over the real
// store, so material order and the ledger are identical to the per-round path.
// Element e of a take that hands out `per` items per element reads items
// [e*per, e*per + per) — the reference's flattened C order.
#include "common.cuh"

#include <stdlib.h>

// local party counts with fused instantiations: every n <= 4, and n = 8
#define FUSED_L_OK(L) (((L) >= 1 && (L) <= 4) || (L) == 8)

#define TAPE_MAX 160  // a whole softmax (rescale, <= 7 tournament levels, attention-exp, reciprocal) fits one tape

struct MatRef {
  const u64* p0;  // triple a | bintriple a | dabit/edabit arithmetic part
  const u64* p1;  // triple b | bintriple b | dabit/edabit bit stream
  const u64* p2;  // triple c | bintriple c
  i64 ps0, ps1, ps2;
  i64 off;        // bit offset of the cursor (bit material)
  int kind;       // 0: arithmetic triple, 1: bit triple, 2: daBit/edaBit
  int per0;       // items per element in p0 (words; bits for kind 1)
  int per1;       // bits per element in p1 (kind 2)
  int pad;
};

struct Tape {
  MatRef m[TAPE_MAX];
  int n;
};

#ifndef MPX_CMP_MINB
#define MPX_CMP_MINB 6  // 80 regs: 1.46 vs 1.63 ms (3 parties, 2^22 ReLU)
#endif

// min resident CTAs per SM (register cap) by local party count: L <= 2 / 3 / 4
#ifndef MPX_MINB3  // L = 3 at 128 regs: ReLU 0.87 / max_vec 2.65 / Log 3.35 ms at 2^22 vs 1.04 / 2.75 / 3.60
#define MPX_MINB3 4     // at 80 regs and 0.90 / 2.67 / 3.84 at 168; LeNet n = 3 step 1.564 vs 1.583 ms
#endif
#ifndef MPX_MINB4  // four parties in one lane (forced MPX_SPLIT4=1 layouts): 128 registers, no spills
#define MPX_MINB4 4
#endif
#define MPX_MINB_L(L, B2) ((L) <= 2 ? (B2) : (L) == 3 ? MPX_MINB3 : (L) == 4 ? MPX_MINB4 : 1)
// n = 8 split over two lanes (4 parties per lane): 128-register cap
#ifndef MPX_MINB_SPLIT
#define MPX_MINB_SPLIT 4
#endif
// split Reciprocal / Exp (n = 4 on two lanes, n = 8 on four): resident CTAs per SM
#ifndef MPX_MINB_G4
#define MPX_MINB_G4 6
#endif
// one lane per element: caps at the register counts ptxas picks unconstrained
// (Reciprocal 56/80/96/146, Exp 47/72/128/168 for L = 1..4); a bare
// minBlocks = 1 lets it take 255 and halves occupancy (Reciprocal 2^24 at
// n = 2: 11.1 vs 8.0 ms)
#ifndef MPX_RCP1_MINB2
#define MPX_RCP1_MINB2 6
#endif
#ifndef MPX_EXP1_MINB2
#define MPX_EXP1_MINB2 6
#endif
#define MPX_MINB_RCP1(L) ((L) <= 2 ? MPX_RCP1_MINB2 : (L) == 3 ? 5 : 3)
#define MPX_MINB_EXP1(L) ((L) <= 2 ? MPX_EXP1_MINB2 : (L) == 3 ? 4 : 3)
#define MPX_MINB_LG(L, G, B2) ((G) > 1 && (L) >= 4 ? MPX_MINB_SPLIT : MPX_MINB_L(L, B2))

#ifndef MPX_LOG_MINB
#define MPX_LOG_MINB 6  // 80 regs, 6 blocks: 8.95 vs 9.34 ms at 2^24
#endif

#ifndef MPX_PREFETCH_DIST
#define MPX_PREFETCH_DIST 0
#endif

__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Party split: with G > 1 an element's n = L*G local parties are held by G
// adjacent lanes, L each (lane g of the group holds parties g*L .. g*L+L-1),
// so n = 8 needs 4 shares per value in registers instead of 8. Every opening
// (a sum or XOR over the parties) is finished with a butterfly over the
// group; both lanes of a group run the same element, so the same control
// path. G = 1 is the one-lane-per-element layout.
//
// Bit 4 of the G template argument (G | MPX_STAGED) marks a kernel whose
// material has been staged into shared memory (k_softmax_fused's staged
// variant): material reads then use generic loads instead of the global-only
// __ldcs / __ldg. GS(G) is the lane-group size.
#define MPX_STAGED 16
#ifndef MPX_STAGED_ROLLED
#define MPX_STAGED_ROLLED 1  // staged kernels keep the carry levels rolled (code size / icache)
#endif
#ifndef MPX_ROLL_ALL
#define MPX_ROLL_ALL 0  // every fused kernel rolled (sweeps)
#endif
#define MPX_ROLLED(G) ((((G) & MPX_STAGED) != 0 && MPX_STAGED_ROLLED) || MPX_ROLL_ALL)
#define GS(G) ((G) & 15)

template <int L, int G>
__device__ __forceinline__ int pbase() {
  return GS(G) == 1 ? 0 : (int)(threadIdx.x & (GS(G) - 1)) * L;
}
#define PI(l) ((l) + pbase<L, G>())

template <int G>
__device__ __forceinline__ unsigned gmask() {
  return GS(G) == 1 ? 0xffffffffu : (((1u << GS(G)) - 1u) << ((threadIdx.x & 31) & ~(unsigned)(GS(G) - 1)));
}
template <int G>
__device__ __forceinline__ u64 gsum(u64 v) {
#pragma unroll
  for (int o = 1; o < GS(G); o <<= 1) v += __shfl_xor_sync(gmask<G>(), v, o);
  return v;
}
template <int G>
__device__ __forceinline__ u64 gxor(u64 v) {
#pragma unroll
  for (int o = 1; o < GS(G); o <<= 1) v ^= __shfl_xor_sync(gmask<G>(), v, o);
  return v;
}

// material loads: streaming (evict-first) / read-only cached from HBM, or
// plain generic loads when the kernel staged its material in shared memory
template <int G>
__device__ __forceinline__ u64 ldm(const u64* p) {
  if constexpr ((G & MPX_STAGED) != 0) return *p; else return __ldcs(p);
}
template <int G>
__device__ __forceinline__ u64 ldr(const u64* p) {
  if constexpr ((G & MPX_STAGED) != 0) return *p; else return __ldg(p);
}
template <int G>
__device__ __forceinline__ ulonglong2 ldr2(const ulonglong2* p) {
  if constexpr ((G & MPX_STAGED) != 0) return *p; else return __ldg(p);
}

// element loop with G lanes per element
#define GRID_STRIDE_G(i, n)                                                                   \
  for (i64 i = ((i64)blockIdx.x * blockDim.x + threadIdx.x) / G; i < (n); i += (i64)gridDim.x * blockDim.x / G)

// Pull take `t`'s slice for element e towards L2 (no registers held).
template <int L, int G>
__device__ __forceinline__ void prefetch_take(const MatRef& t, i64 e) {
  if (t.kind == 0) {
#pragma unroll
    for (int l = 0; l < L; ++l) {
      pf_l2(t.p0 + PI(l) * t.ps0 + e);
      pf_l2(t.p1 + PI(l) * t.ps1 + e);
      pf_l2(t.p2 + PI(l) * t.ps2 + e);
    }
  } else if (t.kind == 1) {
    const i64 w = (t.off + e * (i64)t.per0) >> 6;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      pf_l2(t.p0 + PI(l) * t.ps0 + w);
      pf_l2(t.p1 + PI(l) * t.ps1 + w);
      pf_l2(t.p2 + PI(l) * t.ps2 + w);
    }
  } else {
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const u64* row = t.p0 + PI(l) * t.ps0 + e * (i64)t.per0;
      for (int q = 0; q < t.per0; q += 16) pf_l2(row + q);
      if (t.p1) pf_l2(t.p1 + PI(l) * t.ps1 + ((t.off + e * (i64)t.per1) >> 6));
    }
  }
}

// Consume the next tape entry, prefetching the one MPX_PREFETCH_DIST ahead.
template <int L, int G>
__device__ __forceinline__ const MatRef& next_take(const Tape& tape, int& ti, i64 e) {
  if (MPX_PREFETCH_DIST > 0) {
    const int ahead = ti + MPX_PREFETCH_DIST;
    if (ahead < tape.n) prefetch_take<L, G>(tape.m[ahead], e);
  }
  return tape.m[ti++];
}

struct FusedParams {
  int w, p, iters, bias, c;
  int L, p0;
  u64 log2e_p;      // enc(log2 e, w, p)
  u64 bias_2p;      // enc(bias, w, 2p)
  u64 one_p;        // enc(1.0, w, p)
  u64 m1_p;         // enc(-1.0, w, p)
  u64 ln2_p;        // enc(ln 2, w, p)
  u64 coef_p[5];    // enc(c_i, w, p), i = 1..4 (scale_fixed)
  u64 coef0_2p;     // enc(c_0, w, 2p) (add_const at doubled precision)
  int coef_nz[5];
  int pf;           // ReLU / max level: prefetch the element's whole tape to L2 first
};

template <int L>
struct Sh {
  u64 v[L];
};

template <int L, int G>
__device__ __forceinline__ Sh<L> sh_lin(const Sh<L>& a, u64 ka, const Sh<L>& b, u64 kb, u64 c0, int p0, u64 msk) {
  Sh<L> o;
#pragma unroll
  for (int l = 0; l < L; ++l) o.v[l] = (a.v[l] * ka + b.v[l] * kb + (PI(l) == p0 ? c0 : 0ull)) & msk;
  return o;
}

template <int L, int G>
__device__ __forceinline__ Sh<L> sh_scale(const Sh<L>& a, u64 ka, u64 c0, int p0, u64 msk) {
  Sh<L> o;
#pragma unroll
  for (int l = 0; l < L; ++l) o.v[l] = (a.v[l] * ka + (PI(l) == p0 ? c0 : 0ull)) & msk;
  return o;
}

// Beaver mul (basic.py:27-42), triple item e of the take
template <int L, int G>
__device__ __forceinline__ Sh<L> d_mul(const Sh<L>& x, const Sh<L>& y, const MatRef& t, i64 e, int p0, u64 msk) {
  u64 a[L], b[L];
  u64 d = 0, f = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    a[l] = ldm<G>(t.p0 + PI(l) * t.ps0 + e);
    b[l] = ldm<G>(t.p1 + PI(l) * t.ps1 + e);
    d += x.v[l] - a[l];
    f += y.v[l] - b[l];
  }
  d = gsum<G>(d);
  f = gsum<G>(f);
  Sh<L> z;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    u64 v = ldm<G>(t.p2 + PI(l) * t.ps2 + e) + d * b[l] + f * a[l];
    if (PI(l) == p0) v += d * f;
    z.v[l] = v & msk;
  }
  return z;
}

template <int L, int G>
__device__ __forceinline__ Sh<L> d_mul(const Sh<L>& x, const Sh<L>& y, const MatRef& t, i64 e, int p0, u64 msk);
template <int L, int G>
__device__ __forceinline__ Sh<L> d_trunc(const Sh<L>& x, const MatRef& lo, const MatRef* hi, i64 e, int f,
                                         bool sgn, int w, int p0, u64 msk);

// truncate(mul(x, y), f) consuming triple, edaBit(w, f), edaBit(w, w-1-f) in order
template <int L, int G>
__device__ __forceinline__ Sh<L> d_mul_trunc(const Sh<L>& x, const Sh<L>& y, const Tape& tape, int& ti, i64 e,
                                             int f, int w, int p0, u64 msk) {
  const MatRef& tm = next_take<L, G>(tape, ti, e);
  const Sh<L> z = d_mul<L, G>(x, y, tm, e, p0, msk);
  const MatRef& lo = next_take<L, G>(tape, ti, e);
  const MatRef* hi = (w - 1 - f > 0) ? &next_take<L, G>(tape, ti, e) : nullptr;
  return d_trunc<L, G>(z, lo, hi, e, f, true, w, p0, msk);
}

// probabilistic truncation (derived.py:20-70); lo/hi = edaBit(w, f), edaBit(w, w-1-f)
template <int L, int G>
__device__ __forceinline__ Sh<L> d_trunc(const Sh<L>& x, const MatRef& lo, const MatRef* hi, i64 e, int f,
                                         bool sgn, int w, int p0, u64 msk) {
  const u64 bias = sgn ? (1ull << (w - 2)) : 0ull;
  const u64 unbias = sgn ? (1ull << (w - 2 - f)) : 0ull;
  u64 h[L];
  u64 s = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    h[l] = hi ? ldm<G>(hi->p0 + PI(l) * hi->ps0 + e) : 0ull;
    u64 v = x.v[l] + ldm<G>(lo.p0 + PI(l) * lo.ps0 + e) + (h[l] << f);
    if (PI(l) == p0) v += bias;
    s += v;
  }
  s = gsum<G>(s);
  const u64 chi = (s & msk) >> f;
  Sh<L> z;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    u64 v = 0ull - h[l];
    if (PI(l) == p0) v += chi - unbias;
    z.v[l] = v & msk;
  }
  return z;
}

// Kogge-Stone carries over m-bit words (basic.py:98-136), consuming one tape
// entry per level; returns the sum bits P0 ^ (G << 1).
// One Kogge-Stone level (basic.py:98-129): bintriple fields for this level's
// G (and P, unless last) AND gates, opened across the L local parties.
template <int L, int G>
__device__ __forceinline__ void d_carry_level(u64 (&Gk)[L], u64 (&P)[L], int m, int s, const MatRef& t, i64 e,
                                              int p0) {
  const bool last = 2 * s >= m;
  const int W = m - s;
  const int RW = last ? W : 2 * W;
  const u64 hi = low_bits(m) & ~low_bits(s);
  const i64 bit = t.off + e * (i64)RW;
  u64 ag[L], bg[L], ap[L], bp[L];
  u64 dg = 0, eg = 0, dp = 0, ep = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    ag[l] = load_bits(t.p0 + PI(l) * t.ps0, bit, W) << s;
    bg[l] = load_bits(t.p1 + PI(l) * t.ps1, bit, W) << s;
    const u64 left = P[l] & hi;
    dg ^= left ^ ag[l];
    eg ^= ((Gk[l] << s) & hi) ^ bg[l];
    if (!last) {
      ap[l] = load_bits(t.p0 + PI(l) * t.ps0, bit + W, W) << s;
      bp[l] = load_bits(t.p1 + PI(l) * t.ps1, bit + W, W) << s;
      dp ^= left ^ ap[l];
      ep ^= ((P[l] << s) & hi) ^ bp[l];
    }
  }
  dg = gxor<G>(dg);
  eg = gxor<G>(eg);
  if (!last) {
    dp = gxor<G>(dp);
    ep = gxor<G>(ep);
  }
#pragma unroll
  for (int l = 0; l < L; ++l) {
    u64 zg = (load_bits(t.p2 + PI(l) * t.ps2, bit, W) << s) ^ (dg & bg[l]) ^ (eg & ag[l]);
    if (PI(l) == p0) zg ^= dg & eg;
    Gk[l] ^= zg;
    if (!last) {
      u64 zp = (load_bits(t.p2 + PI(l) * t.ps2, bit + W, W) << s) ^ (dp & bp[l]) ^ (ep & ap[l]);
      if (PI(l) == p0) zp ^= dp & ep;
      P[l] = (P[l] & low_bits(s)) | zp;
    }
  }
}

// Kogge-Stone carries over m-bit words (basic.py:98-136), consuming one tape
// entry per level; returns the sum bits P0 ^ (G << 1). m = 64 (the common
// ring) runs as a fully unrolled level sequence so independent loads of the
// next level can be scheduled early.
template <int L, int G>
__device__ __forceinline__ void d_carry_sum(u64 (&Gk)[L], u64 (&P)[L], const u64 (&P0)[L], int m, const Tape& tape,
                                            int& ti, i64 e, int p0, Sh<L>& out) {
  // levels s = 1, 2, 4, ... < m, unrolled; the 64-bit ring gets its own
  // constant-m copy (measured 7.7 vs 8.9 ms for the 2^24 Reciprocal)
  if constexpr (MPX_ROLLED(G)) {
    // staged (latency-bound, single-row) kernels: one rolled copy keeps the
    // chain's code in the instruction cache
#pragma unroll 1
    for (int s = 1; s < m; s *= 2) d_carry_level<L, G>(Gk, P, m, s, next_take<L, G>(tape, ti, e), e, p0);
  } else if (m == 64) {
#pragma unroll
    for (int s = 1; s < 64; s *= 2) d_carry_level<L, G>(Gk, P, 64, s, next_take<L, G>(tape, ti, e), e, p0);
  } else {
#pragma unroll
    for (int s = 1; s < 64; s *= 2)
      if (s < m) d_carry_level<L, G>(Gk, P, m, s, next_take<L, G>(tape, ti, e), e, p0);
  }
#pragma unroll
  for (int l = 0; l < L; ++l) out.v[l] = (P0[l] ^ (Gk[l] << 1)) & low_bits(m);
}

// bit decomposition (basic.py:199-214): edaBit(w, w) then the carry tree
template <int L, int G>
__device__ __forceinline__ Sh<L> d_decompose(const Sh<L>& x, int w, const Tape& tape, int& ti, i64 e, int p0) {
  const MatRef& t = next_take<L, G>(tape, ti, e);
  const u64 msk = ring_mask(w);
  u64 c = 0;
  u64 rb[L];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    c += x.v[l] - ldm<G>(t.p0 + PI(l) * t.ps0 + e);
    rb[l] = load_bits(t.p1 + PI(l) * t.ps1, t.off + e * (i64)w, w);
  }
  c = gsum<G>(c);
  c &= msk;
  u64 Gk[L], P[L], P0[L];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    Gk[l] = rb[l] & c;
    P[l] = (PI(l) == p0) ? (rb[l] ^ c) : rb[l];
    P0[l] = P[l];
  }
  Sh<L> out;
  d_carry_sum<L, G>(Gk, P, P0, w, tape, ti, e, p0, out);
  return out;
}

// one leftmost-one level: suffix OR via a ^ b ^ ab
template <int L, int G>
__device__ __forceinline__ void d_lmo_level(u64 (&Y)[L], int m, int s, const MatRef& t, i64 e, int p0) {
  const int W = m - s;
  const u64 mw = low_bits(W);
  const i64 bit = t.off + e * (i64)W;
  u64 a[L], b[L];
  u64 d = 0, f = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    a[l] = load_bits(t.p0 + PI(l) * t.ps0, bit, W);
    b[l] = load_bits(t.p1 + PI(l) * t.ps1, bit, W);
    d ^= (Y[l] & mw) ^ a[l];
    f ^= ((Y[l] >> s) & mw) ^ b[l];
  }
  d = gxor<G>(d);
  f = gxor<G>(f);
#pragma unroll
  for (int l = 0; l < L; ++l) {
    u64 z = load_bits(t.p2 + PI(l) * t.ps2, bit, W) ^ (d & b[l]) ^ (f & a[l]);
    if (PI(l) == p0) z ^= d & f;
    const u64 lo = Y[l] & mw, hi = (Y[l] >> s) & mw;
    Y[l] = (Y[l] & ~mw) | ((lo ^ hi ^ z) & mw);
  }
}

// leftmost one (derived.py:131-149); levels unrolled like the carries
template <int L, int G>
__device__ __forceinline__ Sh<L> d_lmo(const Sh<L>& bits, int m, const Tape& tape, int& ti, i64 e, int p0) {
  u64 Y[L];
#pragma unroll
  for (int l = 0; l < L; ++l) Y[l] = bits.v[l];
  if constexpr (MPX_ROLLED(G)) {  // one rolled copy (see d_carry_sum)
#pragma unroll 1
    for (int s = 1; s < m; s *= 2) d_lmo_level<L, G>(Y, m, s, next_take<L, G>(tape, ti, e), e, p0);
  } else if (m == 63) {
#pragma unroll
    for (int s = 1; s < 63; s *= 2) d_lmo_level<L, G>(Y, 63, s, next_take<L, G>(tape, ti, e), e, p0);
  } else if (m == 46) {  // Log's 2p window at the default p = 23
#pragma unroll
    for (int s = 1; s < 46; s *= 2) d_lmo_level<L, G>(Y, 46, s, next_take<L, G>(tape, ti, e), e, p0);
  } else {
#pragma unroll
    for (int s = 1; s < 64; s *= 2)
      if (s < m) d_lmo_level<L, G>(Y, m, s, next_take<L, G>(tape, ti, e), e, p0);
  }
  Sh<L> o;
#pragma unroll
  for (int l = 0; l < L; ++l) o.v[l] = Y[l] ^ (Y[l] >> 1);
  return o;
}

// bit2a opening of an m-bit row (basic.py:164-184): returns the opened c word
template <int L, int G>
__device__ __forceinline__ u64 d_bit2a_open(const Sh<L>& b, int m, const MatRef& t, i64 e) {
  u64 c = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) c ^= b.v[l] ^ load_bits(t.p1 + PI(l) * t.ps1, t.off + e * (i64)m, m);
  return gxor<G>(c) & low_bits(m);
}

// converted bit j of the row: r_arith * (1 - 2c_j) + [p0] c_j
template <int L, int G>
__device__ __forceinline__ Sh<L> d_bit2a_get(u64 c, int j, int m, const MatRef& t, i64 e, int p0, u64 msk) {
  const u64 cj = (c >> j) & 1ull;
  Sh<L> z;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    u64 v = ldr<G>(t.p0 + PI(l) * t.ps0 + e * (i64)m + j) * (1ull - 2ull * cj);
    if (PI(l) == p0) v += cj;
    z.v[l] = v & msk;
  }
  return z;
}

// Stream a whole converted row z_0..z_{m-1} (per party) through `f(l, j, z)`.
// Each party's m daBit words are contiguous (items e*m .. e*m+m-1): read them
// with back-to-back 16-byte L1-cached vector loads so every sector is used.
template <int L, int G, class F>
__device__ __forceinline__ void d_bit2a_row(u64 c, int m, int stride, const MatRef& t, i64 e, int p0, u64 msk,
                                            F&& f) {
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const u64* row = t.p0 + PI(l) * t.ps0 + e * (i64)stride;
    int j = 0;
    auto emit = [&](int jj, u64 r) {
      const u64 cj = (c >> jj) & 1ull;
      u64 v = r * (1ull - 2ull * cj);
      if (PI(l) == p0) v += cj;
      f(l, jj, v & msk);
    };
    if (((uintptr_t)row & 15) != 0 && m > 0) {
      emit(0, ldr<G>(row));
      j = 1;
    }
    for (; j + 8 <= m; j += 8) {
      const ulonglong2* r2 = reinterpret_cast<const ulonglong2*>(row + j);
      const ulonglong2 v0 = ldr2<G>(r2), v1 = ldr2<G>(r2 + 1), v2 = ldr2<G>(r2 + 2), v3 = ldr2<G>(r2 + 3);
      emit(j, v0.x); emit(j + 1, v0.y); emit(j + 2, v1.x); emit(j + 3, v1.y);
      emit(j + 4, v2.x); emit(j + 5, v2.y); emit(j + 6, v3.x); emit(j + 7, v3.y);
    }
    for (; j + 2 <= m; j += 2) {
      const ulonglong2 v0 = ldr2<G>(reinterpret_cast<const ulonglong2*>(row + j));
      emit(j, v0.x);
      emit(j + 1, v0.y);
    }
    if (j < m) emit(j, ldr<G>(row + j));
  }
}

// Material of one truncate(mul(x, y), f) step: triple + edaBit(w,f) + edaBit(w,w-1-f).
// Loads are independent of data, so chains of these steps are software
// pipelined: step k+1's material is loaded while step k computes.
template <int L>
struct MTM {
  u64 a[L], b[L], c[L], lo[L], hi[L];
};

template <int L, int G>
__device__ __forceinline__ void mt_load(MTM<L>& m, const Tape& tape, int& ti, i64 e, int f, int w) {
  const MatRef& tm = next_take<L, G>(tape, ti, e);
  const MatRef& lo = next_take<L, G>(tape, ti, e);
  const bool has_hi = w - 1 - f > 0;
  const MatRef* hi = has_hi ? &next_take<L, G>(tape, ti, e) : nullptr;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    m.a[l] = ldm<G>(tm.p0 + PI(l) * tm.ps0 + e);
    m.b[l] = ldm<G>(tm.p1 + PI(l) * tm.ps1 + e);
    m.c[l] = ldm<G>(tm.p2 + PI(l) * tm.ps2 + e);
    m.lo[l] = ldm<G>(lo.p0 + PI(l) * lo.ps0 + e);
    m.hi[l] = hi ? ldm<G>(hi->p0 + PI(l) * hi->ps0 + e) : 0ull;
  }
}

template <int L, int G>
__device__ __forceinline__ Sh<L> mt_compute(const Sh<L>& x, const Sh<L>& y, const MTM<L>& m, int f, int w, int p0,
                                            u64 msk) {
  u64 d = 0, g = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    d += x.v[l] - m.a[l];
    g += y.v[l] - m.b[l];
  }
  d = gsum<G>(d);
  g = gsum<G>(g);
  const u64 bias = 1ull << (w - 2), unbias = 1ull << (w - 2 - f);
  u64 z[L];
  u64 s = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    u64 v = m.c[l] + d * m.b[l] + g * m.a[l];
    if (PI(l) == p0) v += d * g;
    z[l] = v & msk;
    u64 t = z[l] + m.lo[l] + (m.hi[l] << f);
    if (PI(l) == p0) t += bias;
    s += t;
  }
  s = gsum<G>(s);
  const u64 chi = (s & msk) >> f;
  Sh<L> o;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    u64 v = 0ull - m.hi[l];
    if (PI(l) == p0) v += chi - unbias;
    o.v[l] = v & msk;
  }
  return o;
}

// polynomial at precision p (derived.py:86-108), coefficients pre-encoded
template <int L, int G>
__device__ __forceinline__ Sh<L> d_poly4(const Sh<L>& x, const FusedParams& P, const Tape& tape, int& ti, i64 e,
                                         u64 msk) {
#ifdef MPX_POLY_PIPELINED
  MTM<L> A, B;
  mt_load<L, G>(A, tape, ti, e, P.p, P.w);
  mt_load<L, G>(B, tape, ti, e, P.p, P.w);
  const Sh<L> x2 = mt_compute<L, G>(x, x, A, P.p, P.w, P.p0, msk);
  mt_load<L, G>(A, tape, ti, e, P.p, P.w);
  const Sh<L> x3 = mt_compute<L, G>(x2, x, B, P.p, P.w, P.p0, msk);
  const Sh<L> x4 = mt_compute<L, G>(x3, x, A, P.p, P.w, P.p0, msk);
#else
  const Sh<L> x2 = d_mul_trunc<L, G>(x, x, tape, ti, e, P.p, P.w, P.p0, msk);
  const Sh<L> x3 = d_mul_trunc<L, G>(x2, x, tape, ti, e, P.p, P.w, P.p0, msk);
  const Sh<L> x4 = d_mul_trunc<L, G>(x3, x, tape, ti, e, P.p, P.w, P.p0, msk);
#endif
  const MatRef& flo = next_take<L, G>(tape, ti, e);
  const MatRef& fhi = next_take<L, G>(tape, ti, e);
  u64 acc[L];
#pragma unroll
  for (int l = 0; l < L; ++l) acc[l] = 0;
  if (P.coef_nz[1]) {
#pragma unroll
    for (int l = 0; l < L; ++l) acc[l] += x.v[l] * P.coef_p[1];
  }
  if (P.coef_nz[2]) {
#pragma unroll
    for (int l = 0; l < L; ++l) acc[l] += x2.v[l] * P.coef_p[2];
  }
  if (P.coef_nz[3]) {
#pragma unroll
    for (int l = 0; l < L; ++l) acc[l] += x3.v[l] * P.coef_p[3];
  }
  if (P.coef_nz[4]) {
#pragma unroll
    for (int l = 0; l < L; ++l) acc[l] += x4.v[l] * P.coef_p[4];
  }
  Sh<L> a;
#pragma unroll
  for (int l = 0; l < L; ++l) a.v[l] = (acc[l] + (PI(l) == P.p0 ? P.coef0_2p : 0ull)) & msk;
  return d_trunc<L, G>(a, flo, &fhi, e, P.p, true, P.w, P.p0, msk);
}

template <int L, int G>
__device__ __forceinline__ Sh<L> load_sh(const u64* x, i64 n, i64 e) {
  Sh<L> s;
#pragma unroll
  for (int l = 0; l < L; ++l) s.v[l] = __ldcs(x + PI(l) * n + e);
  return s;
}

template <int L, int G>
__device__ __forceinline__ void store_sh(u64* y, i64 n, i64 e, const Sh<L>& s) {
#pragma unroll
  for (int l = 0; l < L; ++l) __stcs(y + PI(l) * n + e, s.v[l]);
}

// ---------------------------------------------------------------------------
// Reciprocal, paper Alg. 1 (nonlinear.py:146-176)

// Reciprocal (Alg. 1, nonlinear.py:146-176) of one element's shares.
template <int L, int G>
__device__ __forceinline__ Sh<L> d_reciprocal(const Sh<L>& x, const Tape& tape, int& ti, i64 e,
                                              const FusedParams& P) {
  const int w = P.w, p = P.p, p0 = P.p0;
  const u64 msk = ring_mask(w);
  const Sh<L> bits = d_decompose<L, G>(x, w, tape, ti, e, p0);
  Sh<L> sign, mag;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    sign.v[l] = (bits.v[l] >> (w - 1)) & 1ull;
    const u64 mm = low_bits(w - 1);
    mag.v[l] = (bits.v[l] & mm) ^ (sign.v[l] ? mm : 0ull);
  }
  const MatRef& tsg = next_take<L, G>(tape, ti, e);
  const u64 csg = d_bit2a_open<L, G>(sign, 1, tsg, e);
  const Sh<L> s = d_bit2a_get<L, G>(csg, 0, 1, tsg, e, p0, msk);
  const Sh<L> sx = d_mul<L, G>(s, x, next_take<L, G>(tape, ti, e), e, p0, msk);
  const Sh<L> x_pos = sh_lin<L, G>(x, 1, sx, 0ull - 2ull, 0, p0, msk);
  const Sh<L> onehot = d_lmo<L, G>(mag, w - 1, tape, ti, e, p0);
  // reversed low 2p window -> compose (basic.py:187-196)
  Sh<L> window;
#pragma unroll
  for (int l = 0; l < L; ++l) window.v[l] = __brevll(onehot.v[l] & low_bits(2 * p)) >> (64 - 2 * p);
  const MatRef& tc = next_take<L, G>(tape, ti, e);
  const u64 cw = d_bit2a_open<L, G>(window, 2 * p, tc, e);
  Sh<L> t;
#pragma unroll
  for (int l = 0; l < L; ++l) t.v[l] = 0;
  d_bit2a_row<L, G>(cw, 2 * p, 2 * p, tc, e, p0, msk, [&](int l, int j, u64 z) { t.v[l] += z << j; });
#pragma unroll
  for (int l = 0; l < L; ++l) t.v[l] &= msk;
  // z = trunc(t * x_pos), Newton product (nonlinear.py:134-143), y = trunc(t * acc):
  // a chain of 2*iters mul+trunc steps, pipelined one step ahead (A/B)
  MTM<L> A, B;
  mt_load<L, G>(A, tape, ti, e, p, w);
  mt_load<L, G>(B, tape, ti, e, p, w);
  const Sh<L> z = mt_compute<L, G>(t, x_pos, A, p, w, p0, msk);
  Sh<L> q = sh_scale<L, G>(z, 0ull - 1ull, P.one_p, p0, msk);
  Sh<L> acc = sh_scale<L, G>(q, 1, P.one_p, p0, msk);
  for (int it = 1; it < P.iters; ++it) {
    mt_load<L, G>(A, tape, ti, e, p, w);
    q = mt_compute<L, G>(q, q, B, p, w, p0, msk);
    mt_load<L, G>(B, tape, ti, e, p, w);
    acc = mt_compute<L, G>(acc, sh_scale<L, G>(q, 1, P.one_p, p0, msk), A, p, w, p0, msk);
  }
  const Sh<L> yv = mt_compute<L, G>(t, acc, B, p, w, p0, msk);
  const Sh<L> sy = d_mul<L, G>(s, yv, next_take<L, G>(tape, ti, e), e, p0, msk);
  return sh_lin<L, G>(yv, 1, sy, 0ull - 2ull, 0, p0, msk);
}

// Standalone kernel keeps its own copy of the body: through d_reciprocal it
// compiles to 72 registers + spills at L = 2 (8.3 vs 7.9 ms at 2^24).
template <int L, int G>
__global__ void __launch_bounds__(128, G >= 2 ? (L >= 4 ? MPX_MINB_SPLIT : MPX_MINB_G4) : MPX_MINB_RCP1(L)) k_reciprocal_fused(u64* __restrict__ y, const u64* __restrict__ xin, i64 n,
                                                          const __grid_constant__ Tape tape, FusedParams P) {
  const int w = P.w, p = P.p, p0 = P.p0;
  const u64 msk = ring_mask(w);
  GRID_STRIDE_G(e, n) {
    int ti = 0;
    const Sh<L> x = load_sh<L, G>(xin, n, e);
    const Sh<L> bits = d_decompose<L, G>(x, w, tape, ti, e, p0);
    Sh<L> sign, mag;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      sign.v[l] = (bits.v[l] >> (w - 1)) & 1ull;
      const u64 mm = low_bits(w - 1);
      mag.v[l] = (bits.v[l] & mm) ^ (sign.v[l] ? mm : 0ull);
    }
    const MatRef& tsg = next_take<L, G>(tape, ti, e);
    const u64 csg = d_bit2a_open<L, G>(sign, 1, tsg, e);
    const Sh<L> s = d_bit2a_get<L, G>(csg, 0, 1, tsg, e, p0, msk);
    const Sh<L> sx = d_mul<L, G>(s, x, next_take<L, G>(tape, ti, e), e, p0, msk);
    const Sh<L> x_pos = sh_lin<L, G>(x, 1, sx, 0ull - 2ull, 0, p0, msk);
    const Sh<L> onehot = d_lmo<L, G>(mag, w - 1, tape, ti, e, p0);
    // reversed low 2p window -> compose (basic.py:187-196)
    Sh<L> window;
#pragma unroll
    for (int l = 0; l < L; ++l) window.v[l] = __brevll(onehot.v[l] & low_bits(2 * p)) >> (64 - 2 * p);
    const MatRef& tc = next_take<L, G>(tape, ti, e);
    const u64 cw = d_bit2a_open<L, G>(window, 2 * p, tc, e);
    Sh<L> t;
#pragma unroll
    for (int l = 0; l < L; ++l) t.v[l] = 0;
    d_bit2a_row<L, G>(cw, 2 * p, 2 * p, tc, e, p0, msk, [&](int l, int j, u64 z) { t.v[l] += z << j; });
#pragma unroll
    for (int l = 0; l < L; ++l) t.v[l] &= msk;
    // z = trunc(t * x_pos), Newton product (nonlinear.py:134-143), y = trunc(t * acc):
    // a chain of 2*iters mul+trunc steps, pipelined one step ahead (A/B)
    MTM<L> A, B;
    mt_load<L, G>(A, tape, ti, e, p, w);
    mt_load<L, G>(B, tape, ti, e, p, w);
    const Sh<L> z = mt_compute<L, G>(t, x_pos, A, p, w, p0, msk);
    Sh<L> q = sh_scale<L, G>(z, 0ull - 1ull, P.one_p, p0, msk);
    Sh<L> acc = sh_scale<L, G>(q, 1, P.one_p, p0, msk);
    for (int it = 1; it < P.iters; ++it) {
      mt_load<L, G>(A, tape, ti, e, p, w);
      q = mt_compute<L, G>(q, q, B, p, w, p0, msk);
      mt_load<L, G>(B, tape, ti, e, p, w);
      acc = mt_compute<L, G>(acc, sh_scale<L, G>(q, 1, P.one_p, p0, msk), A, p, w, p0, msk);
    }
    const Sh<L> yv = mt_compute<L, G>(t, acc, B, p, w, p0, msk);
    const Sh<L> sy = d_mul<L, G>(s, yv, next_take<L, G>(tape, ti, e), e, p0, msk);
    store_sh<L, G>(y, n, e, sh_lin<L, G>(yv, 1, sy, 0ull - 2ull, 0, p0, msk));
  }
}

// ---------------------------------------------------------------------------
// Exponentiation, paper Alg. 2 (nonlinear.py:179-213)

template <int L, int G>
__global__ void __launch_bounds__(128, G >= 2 ? (L >= 4 ? MPX_MINB_SPLIT : MPX_MINB_G4) : MPX_MINB_EXP1(L)) k_exp_fused(u64* __restrict__ y, const u64* __restrict__ xin, i64 n,
                                                   const __grid_constant__ Tape tape, FusedParams P) {
  const int w = P.w, p = P.p, p0 = P.p0, c = P.c, bias = P.bias;
  const u64 msk = ring_mask(w);
  GRID_STRIDE_G(e, n) {
    int ti = 0;
    if (P.pf)  // small calls are latency-bound: pull the element's whole tape towards L2 first
      for (int i = 0; i < tape.n; ++i) prefetch_take<L, G>(tape.m[i], e);
    const Sh<L> x = load_sh<L, G>(xin, n, e);
    const Sh<L> xb = sh_scale<L, G>(x, P.log2e_p, P.bias_2p, p0, msk);
    const Sh<L> bits = d_decompose<L, G>(xb, w, tape, ti, e, p0);
    const int k = p + c + 1;
    Sh<L> seg;
#pragma unroll
    for (int l = 0; l < L; ++l)
      seg.v[l] = ((bits.v[l] >> p) & low_bits(p + c)) | (((bits.v[l] >> (w - 1)) & 1ull) << (p + c));
    const MatRef& tc = next_take<L, G>(tape, ti, e);
    const u64 cw = d_bit2a_open<L, G>(seg, k, tc, e);
    Sh<L> t;
#pragma unroll
    for (int l = 0; l < L; ++l) t.v[l] = 0;
    // fraction window: first p converted bits, streamed; the row stays in L1
    d_bit2a_row<L, G>(cw, p, k, tc, e, p0, msk, [&](int l, int j, u64 z) { t.v[l] += z << j; });
#pragma unroll
    for (int l = 0; l < L; ++l) t.v[l] &= msk;
    // 2^int as a product of (2^(2^i) b_i - b_i + 1) (nonlinear.py:125-131)
    Sh<L> pw = sh_scale<L, G>(d_bit2a_get<L, G>(cw, p, k, tc, e, p0, msk), 1ull, 1ull, p0, msk);
    for (int i = 1; i < c; ++i) {
      const Sh<L> bi = d_bit2a_get<L, G>(cw, p + i, k, tc, e, p0, msk);
      const u64 kf = (1ull << (1 << i)) - 1ull;
      pw = d_mul<L, G>(pw, sh_scale<L, G>(bi, kf, 1ull, p0, msk), next_take<L, G>(tape, ti, e), e, p0, msk);
    }
    const Sh<L> sgn = d_bit2a_get<L, G>(cw, p + c, k, tc, e, p0, msk);
    const Sh<L> poly = d_poly4<L, G>(t, P, tape, ti, e, msk);
    const Sh<L> yv = d_mul<L, G>(pw, poly, next_take<L, G>(tape, ti, e), e, p0, msk);
    const Sh<L> s1 = sh_scale<L, G>(sgn, 0ull - 1ull, 1ull, p0, msk);
    const Sh<L> out = d_mul_trunc<L, G>(s1, yv, tape, ti, e, bias, w, p0, msk);
    store_sh<L, G>(y, n, e, out);
  }
}

// ---------------------------------------------------------------------------
// Attention exponential 2^x (App. E; nonlinear.py:315-356): narrow w_in = 32
// input decomposed in its own ring, bits converted into the 64-bit ring, the
// fraction evaluated by the square-completed polynomial (nonlinear.py:59-86).
// P.coef_p[0] = enc(p + delta, 32, p), coef_p[1..3] = enc(t3 | t2 | lead*t1,
// 64, p), coef0_2p = enc(lead*t0, 64, 2p), P.bias = lead_shift, P.c = c.

// attention_exp (App. E, nonlinear.py:315-356): narrow input, 64-bit output.
template <int L, int G>
__device__ __forceinline__ Sh<L> d_attexp(const Sh<L>& x, const Tape& tape, int& ti, i64 e, const FusedParams& P) {
  const int win = P.w, p = P.p, p0 = P.p0, c = P.c;
  const u64 msk_in = ring_mask(win), msk = ring_mask(64);
  const Sh<L> xb = sh_scale<L, G>(x, 1ull, P.coef_p[0], p0, msk_in);
  const Sh<L> bits = d_decompose<L, G>(xb, win, tape, ti, e, p0);
  const int k = p + c + 1;
  Sh<L> seg;
#pragma unroll
  for (int l = 0; l < L; ++l)
    seg.v[l] = (bits.v[l] & low_bits(p + c)) | (((bits.v[l] >> (win - 1)) & 1ull) << (p + c));
  const MatRef& tc = next_take<L, G>(tape, ti, e);
  const u64 cw = d_bit2a_open<L, G>(seg, k, tc, e);
  Sh<L> t;
#pragma unroll
  for (int l = 0; l < L; ++l) t.v[l] = 0;
  d_bit2a_row<L, G>(cw, p, k, tc, e, p0, msk, [&](int l, int j, u64 z) { t.v[l] += z << j; });
  // 2^int as a product of (2^(2^i) b_i - b_i + 1) (nonlinear.py:125-131)
  Sh<L> pw = sh_scale<L, G>(d_bit2a_get<L, G>(cw, p, k, tc, e, p0, msk), 1ull, 1ull, p0, msk);
  for (int i = 1; i < c; ++i) {
    const Sh<L> bi = d_bit2a_get<L, G>(cw, p + i, k, tc, e, p0, msk);
    const u64 kf = (1ull << (1 << i)) - 1ull;
    pw = d_mul<L, G>(pw, sh_scale<L, G>(bi, kf, 1ull, p0, msk), next_take<L, G>(tape, ti, e), e, p0, msk);
  }
  const Sh<L> sgn = d_bit2a_get<L, G>(cw, p + c, k, tc, e, p0, msk);
  // evaluate_square_completed (derived.py:111-128)
  const Sh<L> u = sh_scale<L, G>(t, 1ull, P.coef_p[1], p0, msk);
  const Sh<L> u2 = d_mul_trunc<L, G>(u, u, tape, ti, e, p, 64, p0, msk);
  const Sh<L> v = sh_scale<L, G>(u2, 1ull, P.coef_p[2], p0, msk);
  const Sh<L> sq = d_mul<L, G>(v, v, next_take<L, G>(tape, ti, e), e, p0, msk);
  Sh<L> lead = sq;  // truncate(sq, 0) is a copy (derived.py:55-57)
  if (P.bias > 0) {
    const MatRef& lo = next_take<L, G>(tape, ti, e);
    const MatRef* hi = (64 - 1 - P.bias > 0) ? &next_take<L, G>(tape, ti, e) : nullptr;
    lead = d_trunc<L, G>(sq, lo, hi, e, P.bias, true, 64, p0, msk);
  }
  Sh<L> acc = sh_lin<L, G>(lead, 1ull, t, P.coef_p[3], P.coef0_2p, p0, msk);
  Sh<L> ev;
  {
    const MatRef& lo = next_take<L, G>(tape, ti, e);
    const MatRef& hi = next_take<L, G>(tape, ti, e);
    ev = d_trunc<L, G>(acc, lo, &hi, e, p, true, 64, p0, msk);
  }
  const Sh<L> yv = d_mul<L, G>(pw, ev, next_take<L, G>(tape, ti, e), e, p0, msk);
  const Sh<L> s1 = sh_scale<L, G>(sgn, 0ull - 1ull, 1ull, p0, msk);
  const Sh<L> out = d_mul_trunc<L, G>(s1, yv, tape, ti, e, p, 64, p0, msk);
  return out;
}

template <int L, int G>
__global__ void __launch_bounds__(128) k_attexp_fused(u64* __restrict__ y, const u64* __restrict__ xin, i64 n,
                                                      const __grid_constant__ Tape tape, FusedParams P) {
  GRID_STRIDE_G(e, n) {
    int ti = 0;
    if (P.pf)  // small calls are latency-bound: pull the element's whole tape towards L2 first
      for (int i = 0; i < tape.n; ++i) prefetch_take<L, G>(tape.m[i], e);
    const Sh<L> x = load_sh<L, G>(xin, n, e);
    store_sh<L, G>(y, n, e, d_attexp<L, G>(x, tape, ti, e, P));
  }
}

// ---------------------------------------------------------------------------
// Logarithm, paper Alg. 3 without the big-input pre-shift (nonlinear.py:216-267)

template <int L, int G>
__global__ void __launch_bounds__(128, MPX_MINB_LG(L, G, MPX_LOG_MINB)) k_log_fused(u64* __restrict__ y, const u64* __restrict__ xin, i64 n,
                                                   const __grid_constant__ Tape tape, FusedParams P) {
  const int w = P.w, p = P.p, p0 = P.p0;
  const u64 msk = ring_mask(w);
  const int m2 = 2 * p;
  GRID_STRIDE_G(e, n) {
    int ti = 0;
    if (P.pf)  // small calls are latency-bound: pull the element's whole tape towards L2 first
      for (int i = 0; i < tape.n; ++i) prefetch_take<L, G>(tape.m[i], e);
    const Sh<L> x = load_sh<L, G>(xin, n, e);
    const Sh<L> bits = d_decompose<L, G>(x, w, tape, ti, e, p0);
    Sh<L> window;
#pragma unroll
    for (int l = 0; l < L; ++l) window.v[l] = bits.v[l] & low_bits(m2);
    const Sh<L> onehot = d_lmo<L, G>(window, m2, tape, ti, e, p0);
    // paired = AND(window, below) (basic.py:82-95), one bintriple per bit
    const MatRef& ta = next_take<L, G>(tape, ti, e);
    u64 a[L], b[L];
    u64 d = 0, f = 0;
    const i64 bit = ta.off + e * (i64)m2;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      a[l] = load_bits(ta.p0 + PI(l) * ta.ps0, bit, m2);
      b[l] = load_bits(ta.p1 + PI(l) * ta.ps1, bit, m2);
      const u64 below = onehot.v[l] >> 1;
      d ^= window.v[l] ^ a[l];
      f ^= below ^ b[l];
    }
    d = gxor<G>(d);
    f = gxor<G>(f);
    Sh<L> seg;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      u64 z = load_bits(ta.p2 + PI(l) * ta.ps2, bit, m2) ^ (d & b[l]) ^ (f & a[l]);
      if (PI(l) == p0) z ^= d & f;
      const u64 r_bit = (u64)(__popcll(z & low_bits(m2)) & 1);
      seg.v[l] = (onehot.v[l] & low_bits(m2)) | (r_bit << m2);
    }
    const int k = m2 + 1;
    const MatRef& tc = next_take<L, G>(tape, ti, e);
    const u64 cw = d_bit2a_open<L, G>(seg, k, tc, e);
    Sh<L> yl, mm, r;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      yl.v[l] = 0;
      mm.v[l] = 0;
    }
    d_bit2a_row<L, G>(cw, k, k, tc, e, p0, msk, [&](int l, int j, u64 z) {
      if (j < m2) {
        yl.v[l] += z * (u64)(long long)(j - p);
        mm.v[l] += z << (m2 - 1 - j);
      } else {
        r.v[l] = z;
      }
    });
    const Sh<L> xr = d_mul<L, G>(x, r, next_take<L, G>(tape, ti, e), e, p0, msk);
    const Sh<L> doubled = sh_lin<L, G>(x, 2, xr, 0ull - 1ull, 0, p0, msk);
    Sh<L> t = d_mul_trunc<L, G>(doubled, sh_scale<L, G>(mm, 1, 0, p0, msk), tape, ti, e, p, w, p0, msk);
    t = sh_scale<L, G>(t, 1, P.m1_p, p0, msk);
    const Sh<L> yr = d_poly4<L, G>(t, P, tape, ti, e, msk);
    Sh<L> pre;
#pragma unroll
    for (int l = 0; l < L; ++l) pre.v[l] = (yr.v[l] + (yl.v[l] << p) + (r.v[l] << p)) & msk;
    Sh<L> out = sh_scale<L, G>(pre, P.ln2_p, 0, p0, msk);
    {
      const MatRef& lo = next_take<L, G>(tape, ti, e);
      const MatRef& hi = next_take<L, G>(tape, ti, e);
      out = d_trunc<L, G>(out, lo, &hi, e, p, true, w, p0, msk);
    }
    store_sh<L, G>(y, n, e, out);
  }
}

// ---------------------------------------------------------------------------
// ReLU (nn.py:92-97): s = bit2a(gt(x, 0)) = bit2a(sign(0 - x)), y = s * x.
// Also stores s (the converted sign) for the backward pass when s_out != 0.

template <int L, int G>
__global__ void __launch_bounds__(128, MPX_MINB_LG(L, G, MPX_CMP_MINB)) k_relu_fused(u64* __restrict__ y, u64* __restrict__ s_out,
                                                    const u64* __restrict__ xin, i64 n,
                                                    const __grid_constant__ Tape tape, FusedParams P) {
  const int w = P.w, p0 = P.p0;
  const u64 msk = ring_mask(w);
  GRID_STRIDE_G(e, n) {
    int ti = 0;
    if (P.pf)
      for (int i = 0; i < tape.n; ++i) prefetch_take<L, G>(tape.m[i], e);
    const Sh<L> x = load_sh<L, G>(xin, n, e);
    Sh<L> diff;
#pragma unroll
    for (int l = 0; l < L; ++l) diff.v[l] = (0ull - x.v[l]) & msk;   // public zero (party 0) - x
    const Sh<L> bits = d_decompose<L, G>(diff, w, tape, ti, e, p0);
    Sh<L> sign;
#pragma unroll
    for (int l = 0; l < L; ++l) sign.v[l] = (bits.v[l] >> (w - 1)) & 1ull;
    const MatRef& tb = next_take<L, G>(tape, ti, e);
    const u64 c = d_bit2a_open<L, G>(sign, 1, tb, e);
    const Sh<L> sa = d_bit2a_get<L, G>(c, 0, 1, tb, e, p0, msk);
    const Sh<L> out = d_mul<L, G>(sa, x, next_take<L, G>(tape, ti, e), e, p0, msk);
    store_sh<L, G>(y, n, e, out);
    if (s_out) store_sh<L, G>(s_out, n, e, sa);
  }
}

// One max_vec tournament level (derived.py:152-170) on pairs (u, v):
// b = gt(u, v) (sign of v - u), s = bit2a(b), winner = v + s * (u - v).
template <int L, int G>
__device__ __forceinline__ Sh<L> d_maxpair(const Sh<L>& u, const Sh<L>& v, const Tape& tape, int& ti, i64 e, int w,
                                           int p0, u64 msk) {
  Sh<L> diff, uv;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    diff.v[l] = (v.v[l] - u.v[l]) & msk;
    uv.v[l] = (u.v[l] - v.v[l]) & msk;
  }
  const Sh<L> bits = d_decompose<L, G>(diff, w, tape, ti, e, p0);
  Sh<L> sign;
#pragma unroll
  for (int l = 0; l < L; ++l) sign.v[l] = (bits.v[l] >> (w - 1)) & 1ull;
  const MatRef& tb = next_take<L, G>(tape, ti, e);
  const u64 c = d_bit2a_open<L, G>(sign, 1, tb, e);
  const Sh<L> sa = d_bit2a_get<L, G>(c, 0, 1, tb, e, p0, msk);
  const Sh<L> m = d_mul<L, G>(sa, uv, next_take<L, G>(tape, ti, e), e, p0, msk);
  Sh<L> out;
#pragma unroll
  for (int l = 0; l < L; ++l) out.v[l] = (v.v[l] + m.v[l]) & msk;
  return out;
}

template <int L, int G>
__global__ void __launch_bounds__(128, MPX_MINB_LG(L, G, MPX_CMP_MINB)) k_maxlevel_fused(u64* __restrict__ win, const u64* __restrict__ uin,
                                                        const u64* __restrict__ vin, i64 n,
                                                        const __grid_constant__ Tape tape, FusedParams P) {
  const int w = P.w, p0 = P.p0;
  const u64 msk = ring_mask(w);
  GRID_STRIDE_G(e, n) {
    int ti = 0;
    if (P.pf)
      for (int i = 0; i < tape.n; ++i) prefetch_take<L, G>(tape.m[i], e);
    const Sh<L> u = load_sh<L, G>(uin, n, e);
    const Sh<L> v = load_sh<L, G>(vin, n, e);
    store_sh<L, G>(win, n, e, d_maxpair<L, G>(u, v, tape, ti, e, w, p0, msk));
  }
}

// The whole max_vec tournament of a row in one CTA (derived.py:152-170): the
// row's values sit in shared memory; level by level, thread j < half plays
// pair (j, half + j) with the level's takes at element e = row * half + j
// (the per-level kernel's flat index, so material use is identical), and an
// odd leftover moves down behind the winners. One launch per max_vec instead
// of one per level (7 for the attention's 128-wide rows).
struct TourLevels {
  int start[17];  // tape index of each level's first take; start[nlev] = tape.n
  int nlev;
};

template <int L, int G>
__global__ void __launch_bounds__(256 * G) k_maxtour_fused(u64* __restrict__ out, const u64* __restrict__ in, i64 rows,
                                                       int d0, const __grid_constant__ Tape tape,
                                                       const __grid_constant__ TourLevels lv, FusedParams P) {
  extern __shared__ u64 vals[];  // [L][d0]
  const int w = P.w, p0 = P.p0;
  const u64 msk = ring_mask(w);
  for (i64 row = blockIdx.x; row < rows; row += gridDim.x) {
    for (int c = threadIdx.x; c < d0; c += blockDim.x)
#pragma unroll
      for (int l = 0; l < L * G; ++l) vals[l * d0 + c] = in[((i64)l * rows + row) * d0 + c];
    __syncthreads();
    int d = d0;
    // lanes j*G .. j*G+G-1 play pair j (blockDim >= G * d0 / 2), each for its L parties
    const int j = threadIdx.x / G;
    for (int lev = 0; lev < lv.nlev; ++lev) {
      const int half = d / 2;
      const int rest = d - 2 * half;
      Sh<L> win;
      if (j < half) {
        int ti = lv.start[lev];
        const i64 e = row * (i64)half + j;
        if (P.pf)
          for (int i = lv.start[lev]; i < lv.start[lev + 1]; ++i) prefetch_take<L, G>(tape.m[i], e);
        Sh<L> u, v;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          u.v[l] = vals[PI(l) * d0 + j];
          v.v[l] = vals[PI(l) * d0 + half + j];
        }
        win = d_maxpair<L, G>(u, v, tape, ti, e, w, p0, msk);
      }
      Sh<L> rv;
      if (j == 0 && rest)
#pragma unroll
        for (int l = 0; l < L; ++l) rv.v[l] = vals[PI(l) * d0 + 2 * half];
      __syncthreads();
      if (j < half)
#pragma unroll
        for (int l = 0; l < L; ++l) vals[PI(l) * d0 + j] = win.v[l];
      if (j == 0 && rest)
#pragma unroll
        for (int l = 0; l < L; ++l) vals[PI(l) * d0 + half] = rv.v[l];
      __syncthreads();
      d = half + rest;
    }
    if (j == 0)
#pragma unroll
      for (int l = 0; l < L; ++l) out[(i64)PI(l) * rows + row] = vals[PI(l) * d0];
    __syncthreads();
  }
}

// softmax_parts (nn.py:115-136) of a row in one CTA: [rescale x = trunc(x *
// log2 e)], narrow to 32 bits, the max_vec tournament, x - max - 1 ulp,
// attention_exp per element, the row sum and its reciprocal. Every stage
// reads its takes at the flat index its standalone kernel uses (rescale /
// exp: row * d0 + j, tournament level: row * half + j, reciprocal: row), and
// the stages' tapes are scheduled with the standalone keys in the standalone
// order, so shares, material use and the ledger equal the per-op path.
struct SoftmaxSegs {
  int resc;        // tape index of the rescale truncation (-1: base-2 input)
  int lev[17];     // tournament level starts
  int nlev;
  int attexp, recip, end;
  u64 log2e_p;     // enc(log2 e, 64, p) for the rescale
  int p, w32;
};

// One row of softmax_parts. `tape` is the concatenated tape (kernel
// parameter) or its staged shadow in shared memory (G | MPX_STAGED).
template <int L, int G>
__device__ __forceinline__ void softmax_row(i64 row, u64* __restrict__ eout, u64* __restrict__ rout,
                                            const u64* __restrict__ in, i64 rows, int d0, const Tape& tape,
                                            const SoftmaxSegs& sg, const FusedParams& Pm, const FusedParams& Pe,
                                            const FusedParams& Pr, u64* sm_vals, int nreal = 1 << 30) {
  // nreal < L * GS(G): trailing dummy party slots (zero shares, zero staged
  // material) pad n = 3 to four lanes; they never touch global memory
  const int p0 = Pm.p0;
  const u64 m64 = ring_mask(64), m32 = ring_mask(sg.w32);
  const int j = threadIdx.x / GS(G);  // lanes j*G .. j*G+G-1 own column j, L parties each
  const int nw = (blockDim.x + 31) / 32;
  u64* part = sm_vals + L * GS(G) * d0;
  Sh<L> v;
  if (j < d0) {
    const i64 e = row * d0 + j;
#pragma unroll
    for (int l = 0; l < L; ++l) v.v[l] = PI(l) < nreal ? in[((i64)PI(l) * rows + row) * d0 + j] : 0ull;
    if (sg.resc >= 0) {  // truncate(scale_fixed(x, log2 e), p) (derived.py:55-83)
      int ti = sg.resc;
      const Sh<L> sc = sh_scale<L, G>(v, sg.log2e_p, 0ull, p0, m64);
      const MatRef& lo = next_take<L, G>(tape, ti, e);
      const MatRef& hi = next_take<L, G>(tape, ti, e);
      v = d_trunc<L, G>(sc, lo, &hi, e, sg.p, true, 64, p0, m64);
    }
#pragma unroll
    for (int l = 0; l < L; ++l) {
      v.v[l] &= m32;  // narrow (nn.py:68-74)
      sm_vals[PI(l) * d0 + j] = v.v[l];
    }
  }
  __syncthreads();
  // max_vec tournament (derived.py:152-170)
  int d = d0;
  for (int lev = 0; lev < sg.nlev; ++lev) {
    const int half = d / 2, rest = d - 2 * half;
    Sh<L> win;
    if (j < half) {
      int ti = sg.lev[lev];
      Sh<L> u, w;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        u.v[l] = sm_vals[PI(l) * d0 + j];
        w.v[l] = sm_vals[PI(l) * d0 + half + j];
      }
      win = d_maxpair<L, G>(u, w, tape, ti, row * (i64)half + j, sg.w32, p0, m32);
    }
    Sh<L> rv;
    if (j == 0 && rest)
#pragma unroll
      for (int l = 0; l < L; ++l) rv.v[l] = sm_vals[PI(l) * d0 + 2 * half];
    __syncthreads();
    if (j < half)
#pragma unroll
      for (int l = 0; l < L; ++l) sm_vals[PI(l) * d0 + j] = win.v[l];
    if (j == 0 && rest)
#pragma unroll
      for (int l = 0; l < L; ++l) sm_vals[PI(l) * d0 + half] = rv.v[l];
    __syncthreads();
    d = half + rest;
  }
  // x - max - 1 ulp (nn.py:100-112), attention_exp, row sum
  Sh<L> ev;
#pragma unroll
  for (int l = 0; l < L; ++l) ev.v[l] = 0;
  if (j < d0) {
    Sh<L> sh;
#pragma unroll
    for (int l = 0; l < L; ++l) sh.v[l] = (v.v[l] - sm_vals[PI(l) * d0] + (PI(l) == p0 ? m32 : 0ull)) & m32;
    int ti = sg.attexp;
    ev = d_attexp<L, G>(sh, tape, ti, row * (i64)d0 + j, Pe);
#pragma unroll
    for (int l = 0; l < L; ++l)
      if (PI(l) < nreal) eout[((i64)PI(l) * rows + row) * d0 + j] = ev.v[l];
  }
#pragma unroll
  for (int l = 0; l < L; ++l) {
    u64 sum = ev.v[l];
#pragma unroll
    for (int o = 16; o >= GS(G); o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) < GS(G)) part[PI(l) * nw + (threadIdx.x >> 5)] = sum;
  }
  __syncthreads();
  if (j == 0) {
    Sh<L> tot;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      u64 sum = 0;
      for (int q = 0; q < nw; ++q) sum += part[PI(l) * nw + q];
      tot.v[l] = sum & m64;
    }
    int ti = sg.recip;
    const Sh<L> r = d_reciprocal<L, G>(tot, tape, ti, row, Pr);
#pragma unroll
    for (int l = 0; l < L; ++l)
      if (PI(l) < nreal) rout[(i64)PI(l) * rows + row] = r.v[l];
  }
  __syncthreads();
}

template <int L, int G>
__global__ void __launch_bounds__(256 * G) k_softmax_fused(u64* __restrict__ eout, u64* __restrict__ rout,
                                                       const u64* __restrict__ in, i64 rows, int d0,
                                                       const __grid_constant__ Tape tape,
                                                       const __grid_constant__ SoftmaxSegs sg, FusedParams Pm,
                                                       FusedParams Pe, FusedParams Pr) {
  extern __shared__ u64 sm_vals[];  // [L][d0] tournament values, then [L][nwarps] row-sum partials
  for (i64 row = blockIdx.x; row < rows; row += gridDim.x)
    softmax_row<L, G>(row, eout, rout, in, rows, d0, tape, sg, Pm, Pe, Pr, sm_vals);
}

// Staged variant: before each row, the CTA copies every word of material the
// row's chain will read (each take's element range for this row: d0 scores
// for the rescale / attention-exp takes, half of the level for a tournament
// level, one element for the reciprocal) into shared memory with all loads
// in flight at once, and rewrites the tape to point there. The ~100
// dependent rounds of the row then wait on shared-memory latency instead of
// a DRAM / L2 round trip each (LeNet's 128 x 10 softmax: one warp per row).
// Plan (row-independent, built on the host): per take and operand array, the
// element count per row and the staged words per party.
struct StagePlan {
  int cnt[TAPE_MAX];        // elements of this take per row
  int off[TAPE_MAX][3];     // word offset of (take, array) in the stage
  int len[TAPE_MAX][3];     // words per party (0: array unused)
  int words;                // total staged words
  int nparties;             // staged party slots (lanes x parties per lane)
  int nreal;                // real parties; slots beyond hold zeros
};

__device__ __forceinline__ i64 stage_lo(const MatRef& t, int a, i64 e_lo) {
  if (t.kind == 0) return e_lo * (i64)max(1, t.per0);           // one word per element
  if (t.kind == 1) return (t.off + e_lo * (i64)t.per0) >> 6;    // bit triples
  return a == 0 ? e_lo * (i64)t.per0 : (t.off + e_lo * (i64)t.per1) >> 6;   // daBit / edaBit
}

template <int L, int G>
__global__ void __launch_bounds__(256 * G) k_softmax_staged(u64* __restrict__ eout, u64* __restrict__ rout,
                                                        const u64* __restrict__ in, i64 rows, int d0,
                                                        const __grid_constant__ Tape tape,
                                                        const __grid_constant__ SoftmaxSegs sg, FusedParams Pm,
                                                        FusedParams Pe, FusedParams Pr,
                                                        const __grid_constant__ StagePlan plan) {
  extern __shared__ __align__(16) u64 smem_all[];
  Tape& st = *reinterpret_cast<Tape*>(smem_all);
  u64* stage = smem_all + (sizeof(Tape) + 15) / 16 * 2;
  u64* vals = stage + plan.words;
  for (i64 row = blockIdx.x; row < rows; row += gridDim.x) {
    // shadow tape: same entries, operand pointers into the stage
    for (int ti = threadIdx.x; ti < tape.n; ti += blockDim.x) {
      MatRef m = tape.m[ti];
      const i64 e_lo = row * plan.cnt[ti];
      const u64** ps[3] = {&m.p0, &m.p1, &m.p2};
      i64* strides[3] = {&m.ps0, &m.ps1, &m.ps2};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (plan.len[ti][a] == 0) continue;
        *ps[a] = stage + plan.off[ti][a] - stage_lo(m, a, e_lo);
        *strides[a] = plan.len[ti][a];
      }
      st.m[ti] = m;
    }
    if (threadIdx.x == 0) st.n = tape.n;
    // copy: thread t takes segments (take, array, party) t, t + blockDim, ...
    // and issues one asynchronous 8-byte copy per word (cp.async: nothing
    // waits until every copy of the row is in flight)
    const int nseg = tape.n * 3 * plan.nparties;
    for (int q = threadIdx.x; q < nseg; q += blockDim.x) {
      const int l = q % plan.nparties, ta = q / plan.nparties, ti = ta / 3, a = ta % 3;
      const int len = plan.len[ti][a];
      if (len == 0) continue;
      const MatRef& m = tape.m[ti];
      const u64* src = a == 0 ? m.p0 : (a == 1 ? m.p1 : m.p2);
      const i64 sps = a == 0 ? m.ps0 : (a == 1 ? m.ps1 : m.ps2);
      const bool real = l < plan.nreal;              // dummy slots: zero fill (no global read)
      src += (real ? l * sps : 0) + stage_lo(m, a, row * plan.cnt[ti]);
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(stage + plan.off[ti][a] + l * len);
      const uint32_t nb = real ? 8u : 0u;
      for (int i = 0; i < len; ++i)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst + 8 * i), "l"(src + i), "r"(nb)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
    __syncthreads();
    softmax_row<L, G | MPX_STAGED>(row, eout, rout, in, rows, d0, st, sg, Pm, Pe, Pr, vals, plan.nreal);
  }
}

extern "C" int mpx_softmax_fused(uint64_t* e_out, uint64_t* r_out, const uint64_t* x, int64_t rows, int d0,
                                 const void* tape_host, const void* segs_host, const void* pm_host,
                                 const void* pe_host, const void* pr_host, void* stream) {
  CHECK_ARG(e_out && r_out && x && rows >= 0 && d0 >= 2 && d0 <= 256 && tape_host && segs_host && pm_host &&
            pe_host && pr_host);
  const Tape& tp = *(const Tape*)tape_host;
  const SoftmaxSegs& sg = *(const SoftmaxSegs*)segs_host;
  const FusedParams& Pm = *(const FusedParams*)pm_host;
  const FusedParams& Pe = *(const FusedParams*)pe_host;
  const FusedParams& Pr = *(const FusedParams*)pr_host;
  CHECK_ARG(tp.n >= 1 && tp.n <= TAPE_MAX && sg.nlev >= 1 && sg.nlev <= 16 && FUSED_L_OK(Pm.L));
  if (rows == 0) return MPX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int gl = Pm.L == 8 ? 2 : 1;  // lanes per column: n = 8 splits its parties over two lanes
  const int threads = max(32, ((gl * d0 + 31) / 32) * 32);
  const unsigned g = (unsigned)min(rows, (i64)dev_sms() * 8);
  const size_t sm = (size_t)Pm.L * (d0 + threads / 32) * 8;
  // staged plan: the row's element range per take (segments in tape order)
  static StagePlan plan;
  bool staged = true;
  if (const char* e = getenv("MPX_SOFTMAX_STAGE")) staged = atoi(e) != 0;
  // n = 3: one party per lane, four lanes per column (the fourth a zero
  // dummy), so each lane carries a third of the row chain's arithmetic
  bool split3 = Pm.L == 3;
  if (const char* e = getenv("MPX_SOFTMAX_SPLIT3")) split3 = split3 && atoi(e) != 0;
  const int slots = split3 ? 4 : Pm.L;
  if (staged) {
    int cur = 0;
    for (int ti = 0; ti < tp.n; ++ti) {
      int cnt;
      if (sg.resc >= 0 && ti < sg.lev[0]) cnt = d0;             // rescale truncation
      else if (ti < sg.attexp) {                                 // tournament levels
        int lev = 0;
        while (lev + 1 < sg.nlev && ti >= sg.lev[lev + 1]) ++lev;
        int dd = d0;
        for (int k = 0; k < lev; ++k) dd = dd / 2 + (dd & 1);
        cnt = dd / 2;
      } else if (ti < sg.recip) cnt = d0;                       // attention exp
      else cnt = 1;                                              // row-sum reciprocal
      plan.cnt[ti] = cnt;
      const MatRef& m = tp.m[ti];
      for (int a = 0; a < 3; ++a) {
        const void* ptr = a == 0 ? (const void*)m.p0 : (a == 1 ? (const void*)m.p1 : (const void*)m.p2);
        int len = 0;
        if (ptr) {
          if (m.kind == 0) len = cnt * max(1, m.per0);
          else if (m.kind == 1) len = (int)(((i64)cnt * m.per0 + 63) / 64 + 2);
          else len = a == 0 ? cnt * m.per0 : (int)(((i64)cnt * m.per1 + 63) / 64 + 2);
        }
        plan.off[ti][a] = cur;
        plan.len[ti][a] = len;
        cur += ((len * slots + 1) / 2) * 2;                     // 16-byte aligned regions
      }
    }
    plan.words = cur;
    plan.nparties = slots;                                       // every local party (all lanes)
    plan.nreal = Pm.L;
    // at least four warps per row: the staging copy is spread over every thread
    const int cthreads = split3 ? max(32, ((4 * d0 + 31) / 32) * 32) : threads;
    const int sthreads = max(cthreads, 128);
    const size_t ssm = (sizeof(Tape) + 15) / 16 * 16 + (size_t)cur * 8 + (size_t)slots * (d0 + sthreads / 32) * 8;
    if (ssm > 200 * 1024) staged = false;
    else {
      static size_t attr_set = 0;
      if (ssm > attr_set) {
        const void* fns[] = {(const void*)k_softmax_staged<1, 1>, (const void*)k_softmax_staged<2, 1>,
                             (const void*)k_softmax_staged<3, 1>, (const void*)k_softmax_staged<4, 1>,
                             (const void*)k_softmax_staged<4, 2>, (const void*)k_softmax_staged<1, 4>};
        for (const void* f : fns)
          if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm) != cudaSuccess)
            return MPX_ERR_CUDA;
        attr_set = ssm;
      }
      switch (Pm.L) {
        case 1: k_softmax_staged<1, 1><<<g, sthreads, ssm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr, plan); break;
        case 2: k_softmax_staged<2, 1><<<g, sthreads, ssm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr, plan); break;
        case 3:
          if (split3)
            k_softmax_staged<1, 4><<<g, sthreads, ssm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr, plan);
          else
            k_softmax_staged<3, 1><<<g, sthreads, ssm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr, plan);
          break;
        case 4: k_softmax_staged<4, 1><<<g, sthreads, ssm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr, plan); break;
        default: k_softmax_staged<4, 2><<<g, sthreads, ssm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr, plan); break;
      }
      return launch_status();
    }
  }
  switch (Pm.L) {
    case 1: k_softmax_fused<1, 1><<<g, threads, sm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr); break;
    case 2: k_softmax_fused<2, 1><<<g, threads, sm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr); break;
    case 3: k_softmax_fused<3, 1><<<g, threads, sm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr); break;
    case 4: k_softmax_fused<4, 1><<<g, threads, sm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr); break;
    default: k_softmax_fused<4, 2><<<g, threads, sm, s>>>(e_out, r_out, x, rows, d0, tp, sg, Pm, Pe, Pr); break;
  }
  return launch_status();
}

extern "C" int mpx_fused_softmax_size(int64_t* segs) {
  *segs = sizeof(SoftmaxSegs);
  return MPX_OK;
}

extern "C" int mpx_maxtour_fused(uint64_t* y, const uint64_t* x, int64_t rows, int d0, const void* tape_host,
                                 const void* levels_host, const void* params_host, void* stream) {
  CHECK_ARG(y && x && rows >= 0 && d0 >= 2 && d0 <= 512 && tape_host && levels_host && params_host);
  const Tape& tp = *(const Tape*)tape_host;
  const TourLevels& lv = *(const TourLevels*)levels_host;
  const FusedParams& P = *(const FusedParams*)params_host;
  CHECK_ARG(tp.n >= 1 && tp.n <= TAPE_MAX && lv.nlev >= 1 && lv.nlev <= 16 && FUSED_L_OK(P.L));
  if (rows == 0) return MPX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int gl = P.L == 8 ? 2 : 1;  // lanes per pair: n = 8 splits its parties over two lanes
  const int threads = min(256 * gl, max(32, ((gl * (d0 / 2) + 31) / 32) * 32));
  const unsigned g = (unsigned)min(rows, (i64)dev_sms() * 16);
  const size_t sm = (size_t)P.L * d0 * 8;
  switch (P.L) {
    case 1: k_maxtour_fused<1, 1><<<g, threads, sm, s>>>(y, x, rows, d0, tp, lv, P); break;
    case 2: k_maxtour_fused<2, 1><<<g, threads, sm, s>>>(y, x, rows, d0, tp, lv, P); break;
    case 3: k_maxtour_fused<3, 1><<<g, threads, sm, s>>>(y, x, rows, d0, tp, lv, P); break;
    case 4: k_maxtour_fused<4, 1><<<g, threads, sm, s>>>(y, x, rows, d0, tp, lv, P); break;
    default: k_maxtour_fused<4, 2><<<g, threads, sm, s>>>(y, x, rows, d0, tp, lv, P); break;
  }
  return launch_status();
}

// ---------------------------------------------------------------------------


// n = 4 split over two lanes (2 parties each) or one lane per element: the
// per-kernel default `def` is the faster of the two at 2^22 elements
// (Log 5.02 vs 5.51 ms, ReLU 1.48 vs 1.60; Reciprocal / Exp under the
// 80-register cap 4.71 / 3.51 vs 4.75 / 3.51 unsplit); MPX_SPLIT4=0/1 forces
// one layout for A/B runs.
static bool split4(bool def) {
  static const int v = [] {
    const char* e = getenv("MPX_SPLIT4");
    return e ? atoi(e) : -1;
  }();
  return v < 0 ? def : v != 0;
}

// n = 8: lanes per element (2: four parties per lane, 4: two), per-kernel
// default `def` measured at 2^22 elements: Reciprocal 10.6 (4 lanes) vs 16.5
// ms (2), Exp 8.3 vs 10.1, Log 10.2 vs 12.7, ReLU 4.9 vs 3.4 (2 lanes kept;
// one lane per element: 33.6 / 26.1 / 28.6 / 3.9 ms); MPX_SPLIT8=2/4 forces.
static int split8(int def) {
  static const int v = [] {
    const char* e = getenv("MPX_SPLIT8");
    return e ? atoi(e) : 0;
  }();
  return v ? v : def;
}

#define DEFINE_LAUNCH(NAME, KFN, S4, S8)                                                                            \
  extern "C" int NAME(uint64_t* y, const uint64_t* x, int64_t n, const void* tape_host,                    \
                      const void* params_host, void* stream) {                                             \
    CHECK_ARG(y && x && n >= 0 && tape_host && params_host);                                               \
    const Tape& tp = *(const Tape*)tape_host;                                                              \
    const FusedParams& P = *(const FusedParams*)params_host;                                               \
    CHECK_ARG(tp.n >= 1 && tp.n <= TAPE_MAX && P.w >= 8 && P.w <= 64 && FUSED_L_OK(P.L));                 \
    if (n == 0) return MPX_OK;                                                                             \
    cudaStream_t s = (cudaStream_t)stream;                                                                 \
    const unsigned g = grid_for(n, 128);                                                                   \
    switch (P.L) {                                                                                         \
      case 1: KFN<1, 1><<<g, 128, 0, s>>>(y, x, n, tp, P); break;                                             \
      case 2: KFN<2, 1><<<g, 128, 0, s>>>(y, x, n, tp, P); break;                                             \
      case 3: KFN<3, 1><<<g, 128, 0, s>>>(y, x, n, tp, P); break;                                             \
      case 4:                                                                                             \
        if (split4(S4)) KFN<2, 2><<<grid_for(2 * n, 128), 128, 0, s>>>(y, x, n, tp, P);                                   \
        else KFN<4, 1><<<g, 128, 0, s>>>(y, x, n, tp, P);                                                               \
        break;                                             \
      default:  /* n = 8: two lanes per element, 4 parties each */ \
        if (split8(S8) == 4) KFN<2, 4><<<grid_for(4 * n, 128), 128, 0, s>>>(y, x, n, tp, P);                               \
        else KFN<4, 2><<<grid_for(2 * n, 128), 128, 0, s>>>(y, x, n, tp, P);                                            \
        break;                                            \
    }                                                                                                      \
    return launch_status();                                                                                \
  }

DEFINE_LAUNCH(mpx_reciprocal_fused, k_reciprocal_fused, true, 4)

#define DEFINE_LAUNCH2(NAME, KFN, S4, S8, T1, T2)                                                                 \
  extern "C" int NAME(uint64_t* y, T1 a1, T2 a2, int64_t n, const void* tape_host, const void* params_host,   \
                      void* stream) {                                                                      \
    CHECK_ARG(y && a2 && n >= 0 && tape_host && params_host);                                              \
    const Tape& tp = *(const Tape*)tape_host;                                                              \
    const FusedParams& P = *(const FusedParams*)params_host;                                               \
    CHECK_ARG(tp.n >= 1 && tp.n <= TAPE_MAX && P.w >= 8 && P.w <= 64 && FUSED_L_OK(P.L));                 \
    if (n == 0) return MPX_OK;                                                                             \
    cudaStream_t s = (cudaStream_t)stream;                                                                 \
    const unsigned g = grid_for(n, 128);                                                                   \
    switch (P.L) {                                                                                         \
      case 1: KFN<1, 1><<<g, 128, 0, s>>>(y, a1, a2, n, tp, P); break;                                        \
      case 2: KFN<2, 1><<<g, 128, 0, s>>>(y, a1, a2, n, tp, P); break;                                        \
      case 3: KFN<3, 1><<<g, 128, 0, s>>>(y, a1, a2, n, tp, P); break;                                        \
      case 4:                                                                                             \
        if (split4(S4)) KFN<2, 2><<<grid_for(2 * n, 128), 128, 0, s>>>(y, a1, a2, n, tp, P);                                   \
        else KFN<4, 1><<<g, 128, 0, s>>>(y, a1, a2, n, tp, P);                                                               \
        break;                                        \
      default:  /* n = 8: two lanes per element, 4 parties each */ \
        if (split8(S8) == 4) KFN<2, 4><<<grid_for(4 * n, 128), 128, 0, s>>>(y, a1, a2, n, tp, P);                               \
        else KFN<4, 2><<<grid_for(2 * n, 128), 128, 0, s>>>(y, a1, a2, n, tp, P);                                            \
        break;                                       \
    }                                                                                                      \
    return launch_status();                                                                                \
  }

// y, s_out (may be NULL), x
DEFINE_LAUNCH2(mpx_relu_fused, k_relu_fused, true, 2, uint64_t*, const uint64_t*)
// winner, u, v
DEFINE_LAUNCH2(mpx_maxlevel_fused, k_maxlevel_fused, true, 2, const uint64_t*, const uint64_t*)
DEFINE_LAUNCH(mpx_exp_fused, k_exp_fused, true, 4)
DEFINE_LAUNCH(mpx_log_fused, k_log_fused, true, 4)
DEFINE_LAUNCH(mpx_attexp_fused, k_attexp_fused, false, 4)

extern "C" int mpx_fused_tour_size(int64_t* levels) {
  *levels = sizeof(TourLevels);
  return MPX_OK;
}

extern "C" int mpx_fused_abi_sizes(int64_t* matref, int64_t* tape, int64_t* params, int64_t* tape_max) {
  *matref = sizeof(MatRef);
  *tape = sizeof(Tape);
  *params = sizeof(FusedParams);
  *tape_max = TAPE_MAX;
  return MPX_OK;
}
