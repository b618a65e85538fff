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

// 4 consecutive ring elements of a draw: element i = u32[q+2i] | u32[q+2i+1]<<32
__device__ __forceinline__ void draw_elems4(u64 k0, u64 k1, i64 q, u64 (&v)[4]) {
  uint32_t w[8];
  stream_u32<8>(k0, k1, q, 8, w);
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = (u64)w[2 * i] | ((u64)w[2 * i + 1] << 32);
}

// 64 consecutive bit-bytes of a draw starting at u32 index q (64 bytes = 16 u32)
__device__ __forceinline__ u64 draw_bits64(u64 k0, u64 k1, i64 q) {
  uint32_t w[16];
  stream_u32<16>(k0, k1, q, 16, w);
  u64 v = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) v |= byte_lsbs4(w[i]) << (4 * i);
  return v;
}

__global__ void k_philox_elems(u64* __restrict__ out, u64 k0, u64 k1, i64 u32_off, i64 count, u64 msk) {
  const i64 groups = (count + 3) >> 2;
  GRID_STRIDE(g, groups) {
    u64 v[4];
    draw_elems4(k0, k1, u32_off + 8 * g, v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const i64 e = 4 * g + i;
      if (e < count) out[e] = v[i] & msk;
    }
  }
}

__global__ void k_philox_bits(u64* __restrict__ out, u64 k0, u64 k1, i64 u32_off, i64 count) {
  const i64 nw = (count + 63) >> 6;
  GRID_STRIDE(w, nw) {
    u64 v = draw_bits64(k0, k1, u32_off + 16 * w);
    const i64 rem = count - (w << 6);
    if (rem < 64) v &= low_bits((int)rem);
    out[w] = v;
  }
}

extern "C" int mpx_philox_elems(uint64_t* out, uint64_t k0, uint64_t k1, int64_t u32_off, int64_t count,
                                int width, void* stream) {
  CHECK_ARG(out && u32_off >= 0 && count >= 0 && width >= 1 && width <= 64);
  if (count == 0) return MPX_OK;
  k_philox_elems<<<grid_for((count + 3) / 4), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out, k0, k1, u32_off, count, ring_mask(width));
  return launch_status();
}

extern "C" int mpx_philox_bits(uint64_t* out_words, uint64_t k0, uint64_t k1, int64_t u32_off,
                               int64_t count, void* stream) {
  CHECK_ARG(out_words && u32_off >= 0 && count >= 0);
  if (count == 0) return MPX_OK;
  k_philox_bits<<<grid_for((count + 63) / 64), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out_words, k0, k1, u32_off, count);
  return launch_status();
}

// Party p < n-1: draw p ; last party: secret - sum of the n-1 draws.
__global__ void k_deal_share_arith(u64* __restrict__ out, i64 out_ps, const u64* __restrict__ secret,
                                   u64 k0, u64 k1, i64 u32_base, i64 count, int n, int p_lo, int L,
                                   u64 msk) {
  const i64 groups = (count + 3) >> 2;
  const i64 draw_u32 = 2 * count;
  const i64 total = (i64)L * groups;
  GRID_STRIDE(t, total) {
    const int l = (int)(t / groups);
    const i64 g = t - (i64)l * groups;
    const int p = p_lo + l;
    u64 v[4];
    if (p < n - 1) {
      draw_elems4(k0, k1, u32_base + p * draw_u32 + 8 * g, v);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const i64 e = 4 * g + i;
        v[i] = e < count ? secret[e] : 0ull;
      }
      for (int k = 0; k < n - 1; ++k) {
        u64 d[4];
        draw_elems4(k0, k1, u32_base + k * draw_u32 + 8 * g, d);
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] -= d[i] & msk;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const i64 e = 4 * g + i;
      if (e < count) out[l * out_ps + e] = v[i] & msk;
    }
  }
}

__global__ void k_deal_share_bits(u64* __restrict__ out, i64 out_ps, const u64* __restrict__ secret,
                                  u64 k0, u64 k1, i64 u32_base, i64 count, int n, int p_lo, int L) {
  const i64 nw = (count + 63) >> 6;
  const i64 draw_u32 = (count + 3) >> 2;
  const i64 total = (i64)L * nw;
  GRID_STRIDE(t, total) {
    const int l = (int)(t / nw);
    const i64 w = t - (i64)l * nw;
    const int p = p_lo + l;
    u64 v;
    if (p < n - 1) {
      v = draw_bits64(k0, k1, u32_base + p * draw_u32 + 16 * w);
    } else {
      v = secret[w];
      for (int k = 0; k < n - 1; ++k) v ^= draw_bits64(k0, k1, u32_base + k * draw_u32 + 16 * w);
    }
    const i64 rem = count - (w << 6);
    if (rem < 64) v &= low_bits((int)rem);
    out[l * out_ps + w] = v;
  }
}

extern "C" int mpx_deal_share_arith(uint64_t* out, int64_t out_ps, const uint64_t* secret, uint64_t k0,
                                    uint64_t k1, int64_t u32_base, int64_t count, int n, int p_lo, int L,
                                    int width, void* stream) {
  CHECK_ARG(out && u32_base >= 0 && count >= 0 && n >= 1 && p_lo >= 0 && L >= 1 && p_lo + L <= n &&
            width >= 1 && width <= 64);
  CHECK_ARG(secret || p_lo + L < n);
  if (count == 0) return MPX_OK;
  const i64 groups = (count + 3) / 4;
  k_deal_share_arith<<<grid_for((i64)L * groups), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out, out_ps, secret, k0, k1, u32_base, count, n, p_lo, L, ring_mask(width));
  return launch_status();
}

extern "C" int mpx_deal_share_bits(uint64_t* out, int64_t out_ps, const uint64_t* secret_words,
                                   uint64_t k0, uint64_t k1, int64_t u32_base, int64_t count, int n,
                                   int p_lo, int L, void* stream) {
  CHECK_ARG(out && u32_base >= 0 && count >= 0 && n >= 1 && p_lo >= 0 && L >= 1 && p_lo + L <= n);
  CHECK_ARG(secret_words || p_lo + L < n);
  if (count == 0) return MPX_OK;
  const i64 nw = (count + 63) / 64;
  k_deal_share_bits<<<grid_for((i64)L * nw), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out, out_ps, secret_words, k0, k1, u32_base, count, n, p_lo, L);
  return launch_status();
}
