// Trusted dealer on the device (preprocessing.py:121-174, ring.py:124-134,
// sharing.py:124-152).
//
// numpy's Generator.bytes(L) reads ceil(L/4) u32 words from a contiguous
// Philox4x64-10 u32 stream (low half of each raw u64 first). Philox is
// counter based, so any u32 of the stream is computable independently: each
// thread regenerates only the blocks covering its own outputs and writes the
// party shares directly (no byte-stream staging in HBM). The host computes
// every draw's u32 offset in the reference's draw order.
#include "common.cuh"

// NU consecutive u32 of the stream from u32 index q. The block window is
// generated into registers with static indices; the runtime phase q & 7 picks
// one of eight fully unrolled extractions (it is uniform across a launch for
// a given party, so the switch does not diverge).
template <int NU, int OFF>
__device__ __forceinline__ void take_u32(const uint32_t (&buf)[NU + 8], uint32_t (&out)[NU]) {
#pragma unroll
  for (int i = 0; i < NU; ++i) out[i] = buf[i + OFF];
}

template <int NU>
__device__ __forceinline__ void stream_window(u64 k0, u64 k1, i64 q, uint32_t (&out)[NU]) {
  static_assert(NU % 8 == 0, "whole Philox blocks");
  const int off = (int)(q & 7);
  const u64 b0 = (u64)(q >> 3);
  uint32_t buf[NU + 8];
#pragma unroll
  for (int b = 0; b < NU / 8 + 1; ++b) {
    if (b == NU / 8 && off == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) buf[8 * b + j] = 0;
      break;
    }
    const Philox4 r = philox4x64_10(b0 + (u64)b + 1ull, k0, k1);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      buf[8 * b + 2 * j] = (uint32_t)r.v[j];
      buf[8 * b + 2 * j + 1] = (uint32_t)(r.v[j] >> 32);
    }
  }
  switch (off) {
    case 0: take_u32<NU, 0>(buf, out); break;
    case 1: take_u32<NU, 1>(buf, out); break;
    case 2: take_u32<NU, 2>(buf, out); break;
    case 3: take_u32<NU, 3>(buf, out); break;
    case 4: take_u32<NU, 4>(buf, out); break;
    case 5: take_u32<NU, 5>(buf, out); break;
    case 6: take_u32<NU, 6>(buf, out); break;
    default: take_u32<NU, 7>(buf, out); break;
  }
}

// DEAL_E consecutive ring elements of a draw: element i = u32[q+2i] | u32[q+2i+1] << 32.
// A draw whose u32 offset is a multiple of 8 starts on a Philox block: the
// elements are the blocks' raw words (no window, no realignment). The branch
// is uniform across a launch (q % 8 is the draw's base offset % 8).
#define DEAL_E 8
__device__ __forceinline__ void draw_elems(u64 k0, u64 k1, i64 q, u64 (&v)[DEAL_E]) {
  if ((q & 7) == 0) {
    const u64 b0 = (u64)(q >> 3) + 1ull;
    Philox4 r[DEAL_E / 4];
#pragma unroll
    for (int b = 0; b < DEAL_E / 4; ++b) r[b] = philox4x64_10(b0 + (u64)b, k0, k1);
#pragma unroll
    for (int b = 0; b < DEAL_E / 4; ++b)
#pragma unroll
      for (int i = 0; i < 4; ++i) v[4 * b + i] = r[b].v[i];
    return;
  }
  uint32_t w[2 * DEAL_E];
  stream_window<2 * DEAL_E>(k0, k1, q, w);
#pragma unroll
  for (int i = 0; i < DEAL_E; ++i) v[i] = (u64)w[2 * i] | ((u64)w[2 * i + 1] << 32);
}

// LSBs of the 8 bytes of x (stream order: low byte first) -> 8 bits. Per
// u32: (u & 0x01010101) * 0x10204080 moves byte b's bit 0 to bit 28 + b with
// no carries into bits 28..31.
__device__ __forceinline__ u64 lsb8(u64 x) {
  const uint32_t lo = (uint32_t)x & 0x01010101u, hi = (uint32_t)(x >> 32) & 0x01010101u;
  return (u64)(((lo * 0x10204080u) >> 28) | (((hi * 0x10204080u) >> 28) << 4));
}

// DEAL_W words of 64 bit-bytes each (ring.random_bits keeps byte & 1)
#define DEAL_W 2
__device__ __forceinline__ void draw_bits(u64 k0, u64 k1, i64 q, u64 (&v)[DEAL_W]) {
  if ((q & 7) == 0) {  // block-aligned draw: word j = blocks 2j, 2j+1
    const u64 b0 = (u64)(q >> 3) + 1ull;
    Philox4 r[2 * DEAL_W];
#pragma unroll
    for (int b = 0; b < 2 * DEAL_W; ++b) r[b] = philox4x64_10(b0 + (u64)b, k0, k1);
#pragma unroll
    for (int j = 0; j < DEAL_W; ++j) {
      u64 x = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x |= lsb8(r[2 * j].v[i]) << (8 * i);
        x |= lsb8(r[2 * j + 1].v[i]) << (8 * (i + 4));
      }
      v[j] = x;
    }
    return;
  }
  uint32_t w[16 * DEAL_W];
  stream_window<16 * DEAL_W>(k0, k1, q, w);
#pragma unroll
  for (int j = 0; j < DEAL_W; ++j) {
    u64 x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x |= byte_lsbs4(w[16 * j + i]) << (4 * i);
    v[j] = x;
  }
}

// Keys by value, or (dk != nullptr) from a device key slot {k0, k1}: the
// dealer's CUDA graph replays every launch with the slot rewritten per seed.
#define LOAD_DKEY()        \
  if (dk != nullptr) {     \
    k0 = __ldg(dk);        \
    k1 = __ldg(dk + 1);    \
  }

__global__ void k_philox_elems(u64* __restrict__ out, u64 k0, u64 k1, const u64* __restrict__ dk, i64 u32_off,
                               i64 count, u64 msk) {
  LOAD_DKEY();
  const i64 groups = (count + DEAL_E - 1) / DEAL_E;
  GRID_STRIDE(g, groups) {
    u64 v[DEAL_E];
    draw_elems(k0, k1, u32_off + 2 * DEAL_E * g, v);
#pragma unroll
    for (int i = 0; i < DEAL_E; ++i) {
      const i64 e = DEAL_E * g + i;
      if (e < count) out[e] = v[i] & msk;
    }
  }
}

__global__ void k_philox_bits(u64* __restrict__ out, u64 k0, u64 k1, const u64* __restrict__ dk, i64 u32_off,
                              i64 count) {
  LOAD_DKEY();
  const i64 nw = (count + 63) >> 6;
  const i64 groups = (nw + DEAL_W - 1) / DEAL_W;
  GRID_STRIDE(g, groups) {
    u64 v[DEAL_W];
    draw_bits(k0, k1, u32_off + 16 * DEAL_W * g, v);
#pragma unroll
    for (int j = 0; j < DEAL_W; ++j) {
      const i64 w = DEAL_W * g + j;
      if (w >= nw) break;
      const i64 rem = count - (w << 6);
      out[w] = rem < 64 ? (v[j] & low_bits((int)rem)) : v[j];
    }
  }
}

static int philox_elems(uint64_t* out, uint64_t k0, uint64_t k1, const uint64_t* dk, int64_t u32_off,
                        int64_t count, int width, void* stream) {
  CHECK_ARG(out && u32_off >= 0 && count >= 0 && width >= 1 && width <= 64);
  if (count == 0) return MPX_OK;
  k_philox_elems<<<grid_for((count + DEAL_E - 1) / DEAL_E), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out, k0, k1, dk, u32_off, count, ring_mask(width));
  return launch_status();
}

static int philox_bits(uint64_t* out_words, uint64_t k0, uint64_t k1, const uint64_t* dk, int64_t u32_off,
                       int64_t count, void* stream) {
  CHECK_ARG(out_words && u32_off >= 0 && count >= 0);
  if (count == 0) return MPX_OK;
  k_philox_bits<<<grid_for(((count + 63) / 64 + DEAL_W - 1) / DEAL_W), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out_words, k0, k1, dk, u32_off, count);
  return launch_status();
}

extern "C" int mpx_philox_elems(uint64_t* out, uint64_t k0, uint64_t k1, int64_t u32_off, int64_t count,
                                int width, void* stream) {
  return philox_elems(out, k0, k1, nullptr, u32_off, count, width, stream);
}

extern "C" int mpx_philox_bits(uint64_t* out_words, uint64_t k0, uint64_t k1, int64_t u32_off,
                               int64_t count, void* stream) {
  return philox_bits(out_words, k0, k1, nullptr, u32_off, count, stream);
}

extern "C" int mpx_philox_elems_dk(uint64_t* out, const uint64_t* dkey, int64_t u32_off, int64_t count, int width,
                                   void* stream) {
  CHECK_ARG(dkey);
  return philox_elems(out, 0, 0, dkey, u32_off, count, width, stream);
}

extern "C" int mpx_philox_bits_dk(uint64_t* out_words, const uint64_t* dkey, int64_t u32_off, int64_t count,
                                  void* stream) {
  CHECK_ARG(dkey);
  return philox_bits(out_words, 0, 0, dkey, u32_off, count, stream);
}

// Party p < n-1: draw p ; last party: secret - sum of the n-1 draws. One
// thread covers a group for every local party, so each draw is generated
// once even when the last party is local too (sim mode: n-1 draws, not 2(n-1)).
__global__ void k_deal_share_arith(u64* __restrict__ out, i64 out_ps, const u64* __restrict__ secret,
                                   u64 k0, u64 k1, const u64* __restrict__ dk, i64 u32_base, i64 count, int n,
                                   int p_lo, int L, u64 msk) {
  LOAD_DKEY();
  const i64 groups = (count + DEAL_E - 1) / DEAL_E;
  const i64 draw_u32 = 2 * count;
  const bool last_local = p_lo + L == n;
  GRID_STRIDE(g, groups) {
    u64 acc[DEAL_E];
#pragma unroll
    for (int i = 0; i < DEAL_E; ++i) {
      const i64 e = DEAL_E * g + i;
      acc[i] = (last_local && e < count) ? secret[e] : 0ull;
    }
    for (int p = last_local ? 0 : p_lo; p < min(n - 1, p_lo + L); ++p) {
      u64 d[DEAL_E];
      draw_elems(k0, k1, u32_base + p * draw_u32 + 2 * DEAL_E * g, d);
      if (p >= p_lo) {
        u64* o = out + (i64)(p - p_lo) * out_ps;
#pragma unroll
        for (int i = 0; i < DEAL_E; ++i) {
          const i64 e = DEAL_E * g + i;
          if (e < count) o[e] = d[i] & msk;
        }
      }
#pragma unroll
      for (int i = 0; i < DEAL_E; ++i) acc[i] -= d[i] & msk;
    }
    if (last_local) {
      u64* o = out + (i64)(n - 1 - p_lo) * out_ps;
#pragma unroll
      for (int i = 0; i < DEAL_E; ++i) {
        const i64 e = DEAL_E * g + i;
        if (e < count) o[e] = acc[i] & msk;
      }
    }
  }
}

__global__ void k_deal_share_bits(u64* __restrict__ out, i64 out_ps, const u64* __restrict__ secret,
                                  u64 k0, u64 k1, const u64* __restrict__ dk, i64 u32_base, i64 count, int n,
                                  int p_lo, int L) {
  LOAD_DKEY();
  const i64 nw = (count + 63) >> 6;
  const i64 groups = (nw + DEAL_W - 1) / DEAL_W;
  const i64 draw_u32 = (count + 3) >> 2;
  const bool last_local = p_lo + L == n;
  GRID_STRIDE(g, groups) {
    u64 acc[DEAL_W];
#pragma unroll
    for (int j = 0; j < DEAL_W; ++j) {
      const i64 w = DEAL_W * g + j;
      acc[j] = (last_local && w < nw) ? secret[w] : 0ull;
    }
    for (int p = last_local ? 0 : p_lo; p < min(n - 1, p_lo + L); ++p) {
      u64 d[DEAL_W];
      draw_bits(k0, k1, u32_base + p * draw_u32 + 16 * DEAL_W * g, d);
#pragma unroll
      for (int j = 0; j < DEAL_W; ++j) {
        const i64 w = DEAL_W * g + j;
        if (w < nw) {
          const i64 rem = count - (w << 6);
          if (rem < 64) d[j] &= low_bits((int)rem);
          if (p >= p_lo) out[(i64)(p - p_lo) * out_ps + w] = d[j];
          acc[j] ^= d[j];
        }
      }
    }
    if (last_local) {
#pragma unroll
      for (int j = 0; j < DEAL_W; ++j) {
        const i64 w = DEAL_W * g + j;
        if (w < nw) {
          const i64 rem = count - (w << 6);
          out[(i64)(n - 1 - p_lo) * out_ps + w] = rem < 64 ? (acc[j] & low_bits((int)rem)) : acc[j];
        }
      }
    }
  }
}

static int deal_share_arith(uint64_t* out, int64_t out_ps, const uint64_t* secret, uint64_t k0, uint64_t k1,
                            const uint64_t* dk, int64_t u32_base, int64_t count, int n, int p_lo, int L, int width,
                            void* stream) {
  CHECK_ARG(out && u32_base >= 0 && count >= 0 && n >= 1 && p_lo >= 0 && L >= 1 && p_lo + L <= n &&
            width >= 1 && width <= 64);
  CHECK_ARG(secret || p_lo + L < n);
  if (count == 0) return MPX_OK;
  const i64 groups = (count + DEAL_E - 1) / DEAL_E;
  k_deal_share_arith<<<grid_for(groups), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out, out_ps, secret, k0, k1, dk, u32_base, count, n, p_lo, L, ring_mask(width));
  return launch_status();
}

static int deal_share_bits(uint64_t* out, int64_t out_ps, const uint64_t* secret_words, uint64_t k0, uint64_t k1,
                           const uint64_t* dk, int64_t u32_base, int64_t count, int n, int p_lo, int L,
                           void* stream) {
  CHECK_ARG(out && u32_base >= 0 && count >= 0 && n >= 1 && p_lo >= 0 && L >= 1 && p_lo + L <= n);
  CHECK_ARG(secret_words || p_lo + L < n);
  if (count == 0) return MPX_OK;
  const i64 groups = ((count + 63) / 64 + DEAL_W - 1) / DEAL_W;
  k_deal_share_bits<<<grid_for(groups), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out, out_ps, secret_words, k0, k1, dk, u32_base, count, n, p_lo, L);
  return launch_status();
}

extern "C" int mpx_deal_share_arith(uint64_t* out, int64_t out_ps, const uint64_t* secret, uint64_t k0,
                                    uint64_t k1, int64_t u32_base, int64_t count, int n, int p_lo, int L,
                                    int width, void* stream) {
  return deal_share_arith(out, out_ps, secret, k0, k1, nullptr, u32_base, count, n, p_lo, L, width, stream);
}

extern "C" int mpx_deal_share_bits(uint64_t* out, int64_t out_ps, const uint64_t* secret_words,
                                   uint64_t k0, uint64_t k1, int64_t u32_base, int64_t count, int n,
                                   int p_lo, int L, void* stream) {
  return deal_share_bits(out, out_ps, secret_words, k0, k1, nullptr, u32_base, count, n, p_lo, L, stream);
}

extern "C" int mpx_deal_share_arith_dk(uint64_t* out, int64_t out_ps, const uint64_t* secret, const uint64_t* dkey,
                                       int64_t u32_base, int64_t count, int n, int p_lo, int L, int width,
                                       void* stream) {
  CHECK_ARG(dkey);
  return deal_share_arith(out, out_ps, secret, 0, 0, dkey, u32_base, count, n, p_lo, L, width, stream);
}

extern "C" int mpx_deal_share_bits_dk(uint64_t* out, int64_t out_ps, const uint64_t* secret_words,
                                      const uint64_t* dkey, int64_t u32_base, int64_t count, int n, int p_lo, int L,
                                      void* stream) {
  CHECK_ARG(dkey);
  return deal_share_bits(out, out_ps, secret_words, 0, 0, dkey, u32_base, count, n, p_lo, L, stream);
}

// ==========================================================================
// Fused per-kind dealer (preprocessing.py:139-171): ONE launch per material
// key. A thread draws the key's secret values for its group straight from the
// Philox stream at their draw-order offsets, derives the
// dependent ones (c = a*b, c = a & b) in registers, then draws the n-1 share
// values and writes only the local parties' shares (the last party's is the
// secret minus / XOR the draws, sharing.py:124-152). Nothing but the output
// shares touches HBM, so a re-deal is bound by the Philox ALU work (see
// tools/micro/philox_bench.cu for the ceiling) instead of a chain of
// draw -> store -> reload -> share kernels.

// store DEAL_E consecutive elements of a group (masked; tail-checked)
__device__ __forceinline__ void store_group(u64* __restrict__ o, i64 g, const u64 (&v)[DEAL_E], u64 msk, i64 count) {
  const i64 e0 = DEAL_E * g;
  if (e0 + DEAL_E <= count && ((reinterpret_cast<uintptr_t>(o + e0) & 15) == 0)) {
#pragma unroll
    for (int i = 0; i < DEAL_E; i += 2)
      *reinterpret_cast<ulonglong2*>(o + e0 + i) = make_ulonglong2(v[i] & msk, v[i + 1] & msk);
  } else {
#pragma unroll
    for (int i = 0; i < DEAL_E; ++i)
      if (e0 + i < count) o[e0 + i] = v[i] & msk;
  }
}

// Share the group's secrets sec (already masked): party p < n-1 gets its draw
// at u32 offset q_sh + p * du (+ the group's offset), the last party the rest.
__device__ __forceinline__ void share_group_arith(const u64 (&sec)[DEAL_E], u64* __restrict__ out, i64 ps, u64 k0,
                                                  u64 k1, i64 q_sh, i64 du, i64 g, i64 count, int n, int p_lo,
                                                  int L, u64 msk) {
  const bool last_local = p_lo + L == n;
  u64 acc[DEAL_E];
#pragma unroll
  for (int i = 0; i < DEAL_E; ++i) acc[i] = sec[i];
  const int p_end = min(n - 1, p_lo + L);
  for (int p = last_local ? 0 : p_lo; p < p_end; ++p) {
    u64 d[DEAL_E];
    draw_elems(k0, k1, q_sh + p * du + 2 * DEAL_E * g, d);
    if (p >= p_lo) store_group(out + (i64)(p - p_lo) * ps, g, d, msk, count);
#pragma unroll
    for (int i = 0; i < DEAL_E; ++i) acc[i] -= d[i] & msk;
  }
  if (last_local) store_group(out + (i64)(n - 1 - p_lo) * ps, g, acc, msk, count);
}

// bit groups: DEAL_W words of the packed stream (bit t = item t)
__device__ __forceinline__ void share_group_bits(const u64 (&sec)[DEAL_W], u64* __restrict__ out, i64 ps, u64 k0,
                                                 u64 k1, i64 q_sh, i64 du, i64 g, i64 count, int n, int p_lo,
                                                 int L) {
  const bool last_local = p_lo + L == n;
  const i64 nw = (count + 63) >> 6;
  u64 tail[DEAL_W], acc[DEAL_W];
#pragma unroll
  for (int j = 0; j < DEAL_W; ++j) {
    const i64 w = DEAL_W * g + j;
    const i64 rem = count - (w << 6);
    tail[j] = w < nw ? (rem < 64 ? low_bits((int)rem) : ~0ull) : 0ull;
    acc[j] = sec[j] & tail[j];
  }
  const int p_end = min(n - 1, p_lo + L);
  for (int p = last_local ? 0 : p_lo; p < p_end; ++p) {
    u64 d[DEAL_W];
    draw_bits(k0, k1, q_sh + p * du + 16 * DEAL_W * g, d);
#pragma unroll
    for (int j = 0; j < DEAL_W; ++j) {
      d[j] &= tail[j];
      if (p >= p_lo && DEAL_W * g + j < nw) out[(i64)(p - p_lo) * ps + DEAL_W * g + j] = d[j];
      acc[j] ^= d[j];
    }
  }
  if (last_local) {
#pragma unroll
    for (int j = 0; j < DEAL_W; ++j)
      if (DEAL_W * g + j < nw) out[(i64)(n - 1 - p_lo) * ps + DEAL_W * g + j] = acc[j];
  }
}

// triple (preprocessing.py:139-145): a . b . n-1 x a-shares . n-1 x b-shares . n-1 x c-shares
__global__ void __launch_bounds__(MPX_THREADS) k_deal_triple(u64* __restrict__ A, u64* __restrict__ B,
                                                             u64* __restrict__ C, i64 ps, u64 k0, u64 k1,
                                                             const u64* __restrict__ dk, i64 count, int n, int p_lo,
                                                             int L, u64 msk) {
  LOAD_DKEY();
  const i64 groups = (count + DEAL_E - 1) / DEAL_E;
  const i64 du = 2 * count;
  GRID_STRIDE(g, groups) {
    u64 a[DEAL_E], b[DEAL_E], c[DEAL_E];
    draw_elems(k0, k1, 2 * DEAL_E * g, a);
    draw_elems(k0, k1, du + 2 * DEAL_E * g, b);
#pragma unroll
    for (int i = 0; i < DEAL_E; ++i) {
      a[i] &= msk;
      b[i] &= msk;
      c[i] = (a[i] * b[i]) & msk;
    }
    share_group_arith(a, A, ps, k0, k1, 2 * du, du, g, count, n, p_lo, L, msk);
    share_group_arith(b, B, ps, k0, k1, 2 * du + (n - 1) * du, du, g, count, n, p_lo, L, msk);
    share_group_arith(c, C, ps, k0, k1, 2 * du + 2 * (n - 1) * du, du, g, count, n, p_lo, L, msk);
  }
}

// One drawn secret per element at u32 offset q_s (masked to `smsk`: ring
// width, or min(w, m) bits for an edaBit value), optionally stored for a
// consumer (the dealer's A @ B), then shared with draws at q_sh + p * 2count
// (mtriple A / B, preprocessing.py:146-152; edaBit values, :165-170).
__global__ void __launch_bounds__(MPX_THREADS) k_deal_gen_arith(u64* __restrict__ out, i64 ps, u64* __restrict__ sec_out,
                                                                u64 k0, u64 k1, const u64* __restrict__ dk, i64 q_s,
                                                                i64 q_sh, i64 count, int n, int p_lo, int L, u64 smsk,
                                                                u64 msk) {
  LOAD_DKEY();
  const i64 groups = (count + DEAL_E - 1) / DEAL_E;
  GRID_STRIDE(g, groups) {
    u64 s[DEAL_E];
    draw_elems(k0, k1, q_s + 2 * DEAL_E * g, s);
#pragma unroll
    for (int i = 0; i < DEAL_E; ++i) s[i] &= smsk;
    if (sec_out != nullptr) store_group(sec_out, g, s, ~0ull, count);
    share_group_arith(s, out, ps, k0, k1, q_sh, 2 * count, g, count, n, p_lo, L, msk);
  }
}

// bintriple (preprocessing.py:153-159): a bits . b bits . shares of a, b, c = a & b
__global__ void __launch_bounds__(MPX_THREADS) k_deal_bintriple(u64* __restrict__ A, u64* __restrict__ B,
                                                                u64* __restrict__ C, i64 ps, u64 k0, u64 k1,
                                                                const u64* __restrict__ dk, i64 count, int n,
                                                                int p_lo, int L) {
  LOAD_DKEY();
  const i64 nw = (count + 63) >> 6;
  const i64 groups = (nw + DEAL_W - 1) / DEAL_W;
  const i64 du = (count + 3) >> 2;
  GRID_STRIDE(g, groups) {
    u64 a[DEAL_W], b[DEAL_W], c[DEAL_W];
    draw_bits(k0, k1, 16 * DEAL_W * g, a);
    draw_bits(k0, k1, du + 16 * DEAL_W * g, b);
#pragma unroll
    for (int j = 0; j < DEAL_W; ++j) c[j] = a[j] & b[j];
    share_group_bits(a, A, ps, k0, k1, 2 * du, du, g, count, n, p_lo, L);
    share_group_bits(b, B, ps, k0, k1, 2 * du + (n - 1) * du, du, g, count, n, p_lo, L);
    share_group_bits(c, C, ps, k0, k1, 2 * du + 2 * (n - 1) * du, du, g, count, n, p_lo, L);
  }
}

// daBit (preprocessing.py:160-164): r bits . n-1 arith-share draws of r . n-1 bit-share draws.
// Threads [0, ga) take element groups (arithmetic shares), the rest word groups (bit shares).
__global__ void __launch_bounds__(MPX_THREADS) k_deal_dabit(u64* __restrict__ AR, i64 aps, u64* __restrict__ BI,
                                                            i64 bps, u64 k0, u64 k1, const u64* __restrict__ dk,
                                                            i64 count, int n, int p_lo, int L, u64 msk) {
  LOAD_DKEY();
  const i64 ga = (count + DEAL_E - 1) / DEAL_E;
  const i64 nw = (count + 63) >> 6;
  const i64 gb = (nw + DEAL_W - 1) / DEAL_W;
  const i64 qr = (count + 3) >> 2;  // u32 of the r draw
  GRID_STRIDE(t, ga + gb) {
    if (t < ga) {
      uint32_t w[2];
      stream_u32<2>(k0, k1, 2 * t, 2, w);  // bytes 8t .. 8t+7 of the r draw
      u64 s[DEAL_E];
#pragma unroll
      for (int i = 0; i < DEAL_E; ++i) s[i] = (w[i >> 2] >> (8 * (i & 3))) & 1u;
      share_group_arith(s, AR, aps, k0, k1, qr, 2 * count, t, count, n, p_lo, L, msk);
    } else {
      const i64 g = t - ga;
      u64 r[DEAL_W];
      draw_bits(k0, k1, 16 * DEAL_W * g, r);
      share_group_bits(r, BI, bps, k0, k1, qr + (n - 1) * 2 * count, qr, g, count, n, p_lo, L);
    }
  }
}

// edaBit bit shares (preprocessing.py:165-170): the packed bits of the values
// (item e's bit j = flat bit e*m + j) shared with n-1 draws of count*m bytes
// at q_sh. A word group regenerates the values it covers from the value draw
// (u32 offset 0; four values per Philox block, cached across the loop).
__global__ void __launch_bounds__(MPX_THREADS) k_deal_edabit_bits(u64* __restrict__ out, i64 ps, u64 k0, u64 k1,
                                                                  const u64* __restrict__ dk, i64 q_sh, i64 count,
                                                                  int m, u64 smsk, int n, int p_lo, int L) {
  LOAD_DKEY();
  const i64 nbits = count * m;
  const i64 nw = (nbits + 63) >> 6;
  const i64 groups = (nw + DEAL_W - 1) / DEAL_W;
  GRID_STRIDE(g, groups) {
    const i64 t0 = 64 * DEAL_W * g;
    const i64 t1 = min(t0 + 64 * DEAL_W, nbits);
    u64 sec[DEAL_W];
#pragma unroll
    for (int j = 0; j < DEAL_W; ++j) sec[j] = 0;
    i64 cur = -1;
    Philox4 blk;
    for (i64 e = t0 / m; e * m < t1; ++e) {
      const i64 b = e >> 2;  // element e = raw u64 e of the value draw
      if (b != cur) {
        blk = philox4x64_10((u64)b + 1ull, k0, k1);
        cur = b;
      }
      const u64 v = blk.v[e & 3] & smsk;
      const i64 pos = e * m - t0;  // bit position of the value's bit 0 in the window (may be < 0)
#pragma unroll
      for (int j = 0; j < DEAL_W; ++j) {
        const i64 s = pos - 64 * j;  // value bit 0 relative to word j
        if (s >= 64 || s <= -64) continue;
        sec[j] |= s >= 0 ? (v << s) : (v >> (-s));
      }
    }
    share_group_bits(sec, out, ps, k0, k1, q_sh, (nbits + 3) >> 2, g, nbits, n, p_lo, L);
  }
}

#define DEAL_PRE(count_)                                                                  \
  CHECK_ARG(count_ >= 0 && n >= 1 && p_lo >= 0 && L >= 1 && p_lo + L <= n);               \
  if (count_ == 0) return MPX_OK;                                                          \
  cudaStream_t s_ = (cudaStream_t)stream

extern "C" int mpx_deal_triple(uint64_t* a, uint64_t* b, uint64_t* c, int64_t ps, uint64_t k0, uint64_t k1,
                               const uint64_t* dkey, int64_t count, int n, int p_lo, int L, int width, void* stream) {
  CHECK_ARG(a && b && c && width >= 1 && width <= 64);
  DEAL_PRE(count);
  k_deal_triple<<<grid_for((count + DEAL_E - 1) / DEAL_E), MPX_THREADS, 0, s_>>>(a, b, c, ps, k0, k1, dkey, count, n,
                                                                                p_lo, L, ring_mask(width));
  return launch_status();
}

extern "C" int mpx_deal_gen_arith(uint64_t* out, int64_t ps, uint64_t* secret_out, uint64_t k0, uint64_t k1,
                                  const uint64_t* dkey, int64_t q_secret, int64_t q_shares, int64_t count, int n,
                                  int p_lo, int L, int secret_bits, int width, void* stream) {
  CHECK_ARG(out && width >= 1 && width <= 64 && secret_bits >= 1 && q_secret >= 0 && q_shares >= 0);
  DEAL_PRE(count);
  const u64 smsk = ring_mask(width) & low_bits(secret_bits);
  k_deal_gen_arith<<<grid_for((count + DEAL_E - 1) / DEAL_E), MPX_THREADS, 0, s_>>>(
      out, ps, secret_out, k0, k1, dkey, q_secret, q_shares, count, n, p_lo, L, smsk, ring_mask(width));
  return launch_status();
}

extern "C" int mpx_deal_bintriple(uint64_t* a, uint64_t* b, uint64_t* c, int64_t ps, uint64_t k0, uint64_t k1,
                                  const uint64_t* dkey, int64_t count, int n, int p_lo, int L, void* stream) {
  CHECK_ARG(a && b && c);
  DEAL_PRE(count);
  const i64 groups = ((count + 63) / 64 + DEAL_W - 1) / DEAL_W;
  k_deal_bintriple<<<grid_for(groups), MPX_THREADS, 0, s_>>>(a, b, c, ps, k0, k1, dkey, count, n, p_lo, L);
  return launch_status();
}

extern "C" int mpx_deal_dabit(uint64_t* arith, int64_t arith_ps, uint64_t* bit_words, int64_t bit_ps, uint64_t k0,
                              uint64_t k1, const uint64_t* dkey, int64_t count, int n, int p_lo, int L, int width,
                              void* stream) {
  CHECK_ARG(arith && bit_words && width >= 1 && width <= 64);
  DEAL_PRE(count);
  const i64 t = (count + DEAL_E - 1) / DEAL_E + ((count + 63) / 64 + DEAL_W - 1) / DEAL_W;
  k_deal_dabit<<<grid_for(t), MPX_THREADS, 0, s_>>>(arith, arith_ps, bit_words, bit_ps, k0, k1, dkey, count, n, p_lo,
                                                    L, ring_mask(width));
  return launch_status();
}

extern "C" int mpx_deal_edabit_bits(uint64_t* bit_words, int64_t ps, uint64_t k0, uint64_t k1, const uint64_t* dkey,
                                    int64_t q_shares, int64_t count, int m, int width, int n, int p_lo, int L,
                                    void* stream) {
  CHECK_ARG(bit_words && m >= 1 && m <= 64 && width >= 1 && width <= 64 && q_shares >= 0);
  DEAL_PRE(count);
  const i64 groups = ((count * m + 63) / 64 + DEAL_W - 1) / DEAL_W;
  k_deal_edabit_bits<<<grid_for(groups), MPX_THREADS, 0, s_>>>(bit_words, ps, k0, k1, dkey, q_shares, count, m,
                                                                ring_mask(width) & low_bits(m), n, p_lo, L);
  return launch_status();
}

// Philox4x64-10 ALU ceiling probe (the dealer's roofline denominator):
// `blocks` counter blocks, two independent blocks per thread iteration, keys
// in uniform registers, the outputs XOR-folded to one word per thread (no
// memory traffic to speak of). tools/micro/philox_bench.cu measures the same
// loop standalone: ~100 G blocks/s on a B200.
__global__ void __launch_bounds__(256) k_philox_probe(u64* __restrict__ out, u64 k0, u64 k1, i64 blocks) {
  u64 acc = 0;
  const i64 stride = (i64)gridDim.x * blockDim.x * 2;
  for (i64 b = ((i64)blockIdx.x * blockDim.x + threadIdx.x) * 2; b < blocks; b += stride) {
    const Philox4 r0 = philox4x64_10((u64)b + 1ull, k0, k1);
    const Philox4 r1 = philox4x64_10((u64)b + 2ull, k0, k1);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc ^= r0.v[i] ^ r1.v[i];
  }
  out[(i64)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int mpx_philox_probe(uint64_t* out, int64_t out_words, int64_t blocks, void* stream) {
  CHECK_ARG(out && blocks >= 0);
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  const i64 grid = (i64)sms * 8;
  CHECK_ARG(out_words >= grid * 256);
  k_philox_probe<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(out, 0x1234567ull, 0x89abcdefull, blocks);
  return launch_status();
}
