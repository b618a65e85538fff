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

// DEAL_E consecutive ring elements of a draw: element i = u32[q+2i] | u32[q+2i+1] << 32
#define DEAL_E 8
__device__ __forceinline__ void draw_elems(u64 k0, u64 k1, i64 q, u64 (&v)[DEAL_E]) {
  uint32_t w[2 * DEAL_E];
  stream_window<2 * DEAL_E>(k0, k1, q, w);
#pragma unroll
  for (int i = 0; i < DEAL_E; ++i) v[i] = (u64)w[2 * i] | ((u64)w[2 * i + 1] << 32);
}

// DEAL_W words of 64 bit-bytes each (ring.random_bits keeps byte & 1)
#define DEAL_W 2
__device__ __forceinline__ void draw_bits(u64 k0, u64 k1, i64 q, u64 (&v)[DEAL_W]) {
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
