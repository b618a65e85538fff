// Shared device helpers for libmpx (sm_100a).
//
// Conventions (see include/mpx.h):
//  * ring elements live in uint64 words masked to the ring width w;
//  * a share array holds L local parties, party-major, party stride `ps`
//    elements (sim mode: L = n parties on one GPU; party mode: L = 1);
//  * binary shares are row-packed: one uint64 word per row, bit j = logical
//    bit j of that row's trailing axis (m <= 64 bits per row);
//  * dealer bit material is a flat packed bit stream (bit t = item t), so a
//    protocol reads its bintriples/daBits/edaBits as unaligned bit fields at
//    (cursor + row*row_bits);
//  * `p0` is the local slot of party 0 (-1 when party 0 lives elsewhere):
//    public constants are added by party 0 only (sharing.py:99-121).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mpx.h"

typedef uint64_t u64;
typedef int64_t i64;

#define MPX_THREADS 256


__host__ __device__ __forceinline__ u64 ring_mask(int w) {
  return w >= 64 ? ~0ull : ((1ull << w) - 1ull);
}

// low `n` bits set, n in [0, 64]
__host__ __device__ __forceinline__ u64 low_bits(int n) {
  return n >= 64 ? ~0ull : ((1ull << n) - 1ull);
}

// Read `n` (<= 64) bits starting at absolute bit offset `bit` of a packed
// little-endian bit array. Arrays are allocated with one spare word so the
// second read is always in bounds.
__device__ __forceinline__ u64 load_bits(const u64* __restrict__ arr, i64 bit, int n) {
  if (n <= 0) return 0;
  const i64 wi = bit >> 6;
  const int sh = (int)(bit & 63);
  u64 v = arr[wi] >> sh;
  if (sh != 0 && sh + n > 64) v |= arr[wi + 1] << (64 - sh);
  return v & low_bits(n);
}

// SM count of the current device (148 on a B200), queried once per process
static inline int dev_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

static inline unsigned grid_for(i64 n, int threads = MPX_THREADS) {
  i64 b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > (i64)dev_sms() * 16) b = (i64)dev_sms() * 16;
  return (unsigned)b;
}

#define GRID_STRIDE(i, n) \
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (i64)gridDim.x * blockDim.x)

static inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MPX_OK : MPX_ERR_CUDA;
}

#define CHECK_ARG(cond) \
  do {                  \
    if (!(cond)) return MPX_ERR_ARG; \
  } while (0)

// --------------------------------------------------------------------------
// Philox4x64-10, bit-exact with numpy.random.Philox (counter pre-incremented:
// block b uses counter b+1; key = two LE 64-bit words).

struct Philox4 {
  u64 v[4];
};

__device__ __forceinline__ Philox4 philox4x64_10(u64 ctr0, u64 k0, u64 k1) {
  u64 c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const u64 lo0 = 0xD2E7470EE14C6C93ull * c0;
    const u64 hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    const u64 lo1 = 0xCA5A826395121157ull * c2;
    const u64 hi1 = __umul64hi(0xCA5A826395121157ull, c2);
    const u64 n0 = hi1 ^ c1 ^ k0;
    const u64 n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  Philox4 o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

// The numpy byte stream is a contiguous sequence of u32 words (low half of
// each raw u64 first). Fetch `n` consecutive u32 starting at u32 index q0.
template <int NMAX>
__device__ __forceinline__ void stream_u32(u64 k0, u64 k1, i64 q0, int n, uint32_t (&out)[NMAX]) {
  // q -> raw u64 index q>>1 -> block (q>>1)>>2 = q>>3, lane (q>>1)&3, half q&1
  i64 blk = -1;
  Philox4 cur;
  for (int i = 0; i < n; ++i) {
    const i64 q = q0 + i;
    const i64 b = q >> 3;
    if (b != blk) {
      cur = philox4x64_10((u64)b + 1ull, k0, k1);
      blk = b;
    }
    const u64 w = cur.v[(q >> 1) & 3];
    out[i] = (q & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
  }
}

// LSBs of the 4 bytes of a u32 (ring.random_bits keeps byte & 1).
__device__ __forceinline__ u64 byte_lsbs4(uint32_t u) {
  return (u64)((u & 1u) | ((u >> 7) & 2u) | ((u >> 14) & 4u) | ((u >> 21) & 8u));
}
