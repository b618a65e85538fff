// Interactive-protocol kernels: the local halves of every round.
//
// A round = mask kernel (partial opening reduced over the L local parties)
// -> [party mode: NCCL all-reduce / all-gather of the partial] -> finish
// kernel. In sim mode (all parties on this GPU) the *_fused kernels do the
// three steps in one pass: the opening is a register-level reduction.
//
// Reference: protocols/basic.py:27-214, protocols/derived.py:20-149.
#include "common.cuh"

// ==========================================================================
// Beaver multiplication (basic.py:27-42)

__global__ void k_mul_finish(u64* __restrict__ z, const u64* __restrict__ d, const u64* __restrict__ e,
                             const u64* __restrict__ a, const u64* __restrict__ b,
                             const u64* __restrict__ c, i64 t_ps, int L, i64 n, u64 msk, int p0) {
  const i64 total = (i64)L * n;
  GRID_STRIDE(t, total) {
    const i64 l = L == 1 ? 0 : t / n;  // party mode (L = 1): no 64-bit division
    const i64 i = t - l * n;
    const i64 m = l * t_ps + i;
    const u64 dv = d[i], ev = e[i];
    u64 v = c[m] + dv * b[m] + ev * a[m];
    if (l == p0) v += dv * ev;
    z[t] = v & msk;
  }
}

extern "C" int mpx_mul_finish(uint64_t* z, const uint64_t* d, const uint64_t* e, const uint64_t* a,
                              const uint64_t* b, const uint64_t* c, int64_t t_ps, int L, int64_t n,
                              int width, int p0, void* stream) {
  CHECK_ARG(z && d && e && a && b && c && L >= 1 && n >= 0 && width >= 1 && width <= 64);
  if (n == 0) return MPX_OK;
  k_mul_finish<<<grid_for((i64)L * n), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      z, d, e, a, b, c, t_ps, L, n, ring_mask(width), p0);
  return launch_status();
}

template <int LMAX>
__global__ void k_mul_fused(u64* __restrict__ z, const u64* __restrict__ x, const u64* __restrict__ y,
                            const u64* __restrict__ a, const u64* __restrict__ b,
                            const u64* __restrict__ c, i64 t_ps, int L, i64 n, u64 msk, int p0) {
  GRID_STRIDE(i, n) {
    u64 av[LMAX], bv[LMAX];
    u64 dv = 0, ev = 0;
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        av[l] = a[l * t_ps + i];
        bv[l] = b[l * t_ps + i];
        dv += x[l * n + i] - av[l];
        ev += y[l * n + i] - bv[l];
      }
    }
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        u64 v = c[l * t_ps + i] + dv * bv[l] + ev * av[l];
        if (l == p0) v += dv * ev;
        z[l * n + i] = v & msk;
      }
    }
  }
}

// Two elements per thread with 16-byte accesses (every party's array 16-byte
// aligned, n and t_ps even).
template <int LMAX>
__global__ void k_mul_fused2(u64* __restrict__ z, const u64* __restrict__ x, const u64* __restrict__ y,
                             const u64* __restrict__ a, const u64* __restrict__ b,
                             const u64* __restrict__ c, i64 t_ps, int L, i64 n, u64 msk, int p0) {
  typedef ulonglong2 V;
  GRID_STRIDE(i2, n / 2) {
    const i64 i = 2 * i2;
    V av[LMAX], bv[LMAX];
    u64 d0 = 0, d1 = 0, e0 = 0, e1 = 0;
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        av[l] = __ldg(reinterpret_cast<const V*>(a + l * t_ps + i));
        bv[l] = __ldg(reinterpret_cast<const V*>(b + l * t_ps + i));
        const V xv = __ldg(reinterpret_cast<const V*>(x + l * n + i));
        const V yv = __ldg(reinterpret_cast<const V*>(y + l * n + i));
        d0 += xv.x - av[l].x;
        d1 += xv.y - av[l].y;
        e0 += yv.x - bv[l].x;
        e1 += yv.y - bv[l].y;
      }
    }
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        const V cv = __ldg(reinterpret_cast<const V*>(c + l * t_ps + i));
        u64 v0 = cv.x + d0 * bv[l].x + e0 * av[l].x, v1 = cv.y + d1 * bv[l].y + e1 * av[l].y;
        if (l == p0) {
          v0 += d0 * e0;
          v1 += d1 * e1;
        }
        *reinterpret_cast<V*>(z + l * n + i) = make_ulonglong2(v0 & msk, v1 & msk);
      }
    }
  }
}

extern "C" int mpx_mul_fused(uint64_t* z, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                             const uint64_t* b, const uint64_t* c, int64_t t_ps, int L, int64_t n,
                             int width, int p0, void* stream) {
  CHECK_ARG(z && x && y && a && b && c && L >= 1 && L <= 16 && n >= 0 && width >= 1 && width <= 64);
  if (n == 0) return MPX_OK;
  const u64 msk = ring_mask(width);
  cudaStream_t s = (cudaStream_t)stream;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (L <= 4 && n >= 1024 && n % 2 == 0 && t_ps % 2 == 0 && al16(z) && al16(x) && al16(y) && al16(a) && al16(b) &&
      al16(c)) {
    if (L <= 2)
      k_mul_fused2<2><<<grid_for(n / 2), MPX_THREADS, 0, s>>>(z, x, y, a, b, c, t_ps, L, n, msk, p0);
    else
      k_mul_fused2<4><<<grid_for(n / 2), MPX_THREADS, 0, s>>>(z, x, y, a, b, c, t_ps, L, n, msk, p0);
    return launch_status();
  }
  if (L <= 2)
    k_mul_fused<2><<<grid_for(n), MPX_THREADS, 0, s>>>(z, x, y, a, b, c, t_ps, L, n, msk, p0);
  else if (L <= 4)
    k_mul_fused<4><<<grid_for(n), MPX_THREADS, 0, s>>>(z, x, y, a, b, c, t_ps, L, n, msk, p0);
  else if (L <= 8)
    k_mul_fused<8><<<grid_for(n), MPX_THREADS, 0, s>>>(z, x, y, a, b, c, t_ps, L, n, msk, p0);
  else
    k_mul_fused<16><<<grid_for(n), MPX_THREADS, 0, s>>>(z, x, y, a, b, c, t_ps, L, n, msk, p0);
  return launch_status();
}

// ==========================================================================
// Probabilistic truncation (derived.py:20-70). r = r_lo + 2^f r_hi from two
// edaBits (arithmetic parts only); open c = x + r (+ 2^(w-2) bias for the
// signed variant, added by party 0); z = (c >> f) - r_hi (- 2^(w-2-f)).

__device__ __forceinline__ u64 trunc_masked(const u64* __restrict__ x, const u64* __restrict__ r_lo,
                                            i64 lo_ps, const u64* __restrict__ r_hi, i64 hi_ps, int l,
                                            i64 n, i64 i, int f, u64 bias, int p0) {
  u64 v = x[l * n + i] + r_lo[l * lo_ps + i];
  if (r_hi) v += r_hi[l * hi_ps + i] << f;
  if (l == p0) v += bias;
  return v;
}

__global__ void k_trunc_mask(u64* __restrict__ out, const u64* __restrict__ x, const u64* __restrict__ r_lo,
                             i64 lo_ps, const u64* __restrict__ r_hi, i64 hi_ps, int L, i64 n, u64 msk,
                             int f, u64 bias, int p0) {
  GRID_STRIDE(i, n) {
    u64 s = 0;
    for (int l = 0; l < L; ++l) s += trunc_masked(x, r_lo, lo_ps, r_hi, hi_ps, l, n, i, f, bias, p0);
    out[i] = s & msk;
  }
}

__global__ void k_trunc_finish(u64* __restrict__ z, const u64* __restrict__ c, const u64* __restrict__ r_hi,
                               i64 hi_ps, int L, i64 n, u64 msk, int f, u64 unbias, int p0) {
  const i64 total = (i64)L * n;
  GRID_STRIDE(t, total) {
    const i64 l = L == 1 ? 0 : t / n;  // party mode (L = 1): no 64-bit division
    const i64 i = t - l * n;
    u64 v = r_hi ? (0ull - r_hi[l * hi_ps + i]) : 0ull;
    if (l == p0) v += ((c[i] & msk) >> f) - unbias;
    z[t] = v & msk;
  }
}

// Two elements per thread with 16-byte loads and stores when every party's
// array is 16-byte aligned (n even, even party strides): half the memory
// instructions of the element-per-thread loop below.
template <int LMAX>
__global__ void k_trunc_fused2(u64* __restrict__ z, const u64* __restrict__ x, const u64* __restrict__ r_lo,
                               i64 lo_ps, const u64* __restrict__ r_hi, i64 hi_ps, int L, i64 n, u64 msk,
                               int f, u64 bias, u64 unbias, int p0) {
  GRID_STRIDE(i2, n / 2) {
    const i64 i = 2 * i2;
    ulonglong2 hv[LMAX];
    u64 s0 = 0, s1 = 0;
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        hv[l] = r_hi ? __ldg(reinterpret_cast<const ulonglong2*>(r_hi + l * hi_ps + i)) : make_ulonglong2(0, 0);
        const ulonglong2 xv = __ldg(reinterpret_cast<const ulonglong2*>(x + l * n + i));
        const ulonglong2 lv = __ldg(reinterpret_cast<const ulonglong2*>(r_lo + l * lo_ps + i));
        u64 v0 = xv.x + lv.x + (hv[l].x << f), v1 = xv.y + lv.y + (hv[l].y << f);
        if (l == p0) {
          v0 += bias;
          v1 += bias;
        }
        s0 += v0;
        s1 += v1;
      }
    }
    const u64 c0 = (s0 & msk) >> f, c1 = (s1 & msk) >> f;
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        u64 v0 = 0ull - hv[l].x, v1 = 0ull - hv[l].y;
        if (l == p0) {
          v0 += c0 - unbias;
          v1 += c1 - unbias;
        }
        *reinterpret_cast<ulonglong2*>(z + l * n + i) = make_ulonglong2(v0 & msk, v1 & msk);
      }
    }
  }
}

template <int LMAX>
__global__ void k_trunc_fused(u64* __restrict__ z, const u64* __restrict__ x, const u64* __restrict__ r_lo,
                              i64 lo_ps, const u64* __restrict__ r_hi, i64 hi_ps, int L, i64 n, u64 msk,
                              int f, u64 bias, u64 unbias, int p0) {
  GRID_STRIDE(i, n) {
    u64 hv[LMAX];
    u64 s = 0;
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        hv[l] = r_hi ? r_hi[l * hi_ps + i] : 0ull;
        u64 v = x[l * n + i] + r_lo[l * lo_ps + i] + (hv[l] << f);
        if (l == p0) v += bias;
        s += v;
      }
    }
    const u64 chi = (s & msk) >> f;
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        u64 v = 0ull - hv[l];
        if (l == p0) v += chi - unbias;
        z[l * n + i] = v & msk;
      }
    }
  }
}

extern "C" int mpx_trunc_mask(uint64_t* out, const uint64_t* x, const uint64_t* r_lo, int64_t lo_ps,
                              const uint64_t* r_hi, int64_t hi_ps, int L, int64_t n, int width, int f,
                              uint64_t bias, int p0, void* stream) {
  CHECK_ARG(out && x && r_lo && L >= 1 && n >= 0 && width >= 2 && width <= 64 && f >= 1 && f < width);
  if (n == 0) return MPX_OK;
  k_trunc_mask<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, x, r_lo, lo_ps, r_hi, hi_ps, L,
                                                                       n, ring_mask(width), f, bias, p0);
  return launch_status();
}

extern "C" int mpx_trunc_finish(uint64_t* z, const uint64_t* c, const uint64_t* r_hi, int64_t hi_ps,
                                int L, int64_t n, int width, int f, uint64_t unbias, int p0,
                                void* stream) {
  CHECK_ARG(z && c && L >= 1 && n >= 0 && width >= 2 && width <= 64 && f >= 1 && f < width);
  if (n == 0) return MPX_OK;
  k_trunc_finish<<<grid_for((i64)L * n), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      z, c, r_hi, hi_ps, L, n, ring_mask(width), f, unbias, p0);
  return launch_status();
}

extern "C" int mpx_trunc_fused(uint64_t* z, const uint64_t* x, const uint64_t* r_lo, int64_t lo_ps,
                               const uint64_t* r_hi, int64_t hi_ps, int L, int64_t n, int width, int f,
                               uint64_t bias, uint64_t unbias, int p0, void* stream) {
  CHECK_ARG(z && x && r_lo && L >= 1 && L <= 16 && n >= 0 && width >= 2 && width <= 64 && f >= 1 &&
            f < width);
  if (n == 0) return MPX_OK;
  const u64 msk = ring_mask(width);
  cudaStream_t s = (cudaStream_t)stream;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec = n % 2 == 0 && lo_ps % 2 == 0 && (r_hi == nullptr || hi_ps % 2 == 0) && al16(z) && al16(x) &&
                   al16(r_lo) && (r_hi == nullptr || al16(r_hi)) && n >= 1024;
  if (vec && L <= 4) {
    if (L <= 2)
      k_trunc_fused2<2><<<grid_for(n / 2), MPX_THREADS, 0, s>>>(z, x, r_lo, lo_ps, r_hi, hi_ps, L, n, msk, f, bias,
                                                                unbias, p0);
    else
      k_trunc_fused2<4><<<grid_for(n / 2), MPX_THREADS, 0, s>>>(z, x, r_lo, lo_ps, r_hi, hi_ps, L, n, msk, f, bias,
                                                                unbias, p0);
    return launch_status();
  }
  if (L <= 2)
    k_trunc_fused<2><<<grid_for(n), MPX_THREADS, 0, s>>>(z, x, r_lo, lo_ps, r_hi, hi_ps, L, n, msk, f,
                                                         bias, unbias, p0);
  else if (L <= 4)
    k_trunc_fused<4><<<grid_for(n), MPX_THREADS, 0, s>>>(z, x, r_lo, lo_ps, r_hi, hi_ps, L, n, msk, f,
                                                         bias, unbias, p0);
  else if (L <= 8)
    k_trunc_fused<8><<<grid_for(n), MPX_THREADS, 0, s>>>(z, x, r_lo, lo_ps, r_hi, hi_ps, L, n, msk, f,
                                                         bias, unbias, p0);
  else
    k_trunc_fused<16><<<grid_for(n), MPX_THREADS, 0, s>>>(z, x, r_lo, lo_ps, r_hi, hi_ps, L, n, msk, f,
                                                          bias, unbias, p0);
  return launch_status();
}

// Several independent sim-mode truncations in ONE launch, each optionally
// subtracted from a base: z = base - trunc(x) (the SGD update W -= trunc(dW)
// of every layer; derived.py:20-70 per job, material in job order).
#define TRUNC_JOBS_MAX 16
struct TruncJob {
  u64* z;
  const u64* base;  // may be null: z = trunc(x)
  const u64* x;
  const u64* r_lo;
  const u64* r_hi;  // may be null (f = w - 1)
  i64 lo_ps, hi_ps, n;
  u64 bias, unbias;
  int f, pad;
};
struct TruncJobs {
  TruncJob j[TRUNC_JOBS_MAX];
  i64 start[TRUNC_JOBS_MAX + 1];  // first block of each job
  int n, pad;
};

template <int LMAX>
__global__ void __launch_bounds__(256) k_trunc_sub_multi(const __grid_constant__ TruncJobs jobs, int L, u64 msk,
                                                         int p0) {
  int k = 0;
  while (k + 1 < jobs.n && (i64)blockIdx.x >= jobs.start[k + 1]) ++k;
  const TruncJob& J = jobs.j[k];
  const i64 i = ((i64)blockIdx.x - jobs.start[k]) * blockDim.x + threadIdx.x;
  if (i >= J.n) return;
  u64 hv[LMAX];
  u64 s = 0;
#pragma unroll
  for (int l = 0; l < LMAX; ++l) {
    if (l < L) {
      hv[l] = J.r_hi ? J.r_hi[l * J.hi_ps + i] : 0ull;
      u64 v = J.x[l * J.n + i] + J.r_lo[l * J.lo_ps + i] + (hv[l] << J.f);
      if (l == p0) v += J.bias;
      s += v;
    }
  }
  const u64 chi = (s & msk) >> J.f;
#pragma unroll
  for (int l = 0; l < LMAX; ++l) {
    if (l < L) {
      u64 v = 0ull - hv[l];
      if (l == p0) v += chi - J.unbias;
      if (J.base) v = J.base[l * J.n + i] - v;
      J.z[l * J.n + i] = v & msk;
    }
  }
}

extern "C" int mpx_trunc_sub_multi(const void* jobs_host, int L, int width, int p0, void* stream) {
  CHECK_ARG(jobs_host && L >= 1 && L <= 16 && width >= 2 && width <= 64);
  TruncJobs J = *(const TruncJobs*)jobs_host;
  CHECK_ARG(J.n >= 1 && J.n <= TRUNC_JOBS_MAX);
  i64 b = 0;
  for (int k = 0; k < J.n; ++k) {
    CHECK_ARG(J.j[k].z && J.j[k].x && J.j[k].r_lo && J.j[k].n >= 0 && J.j[k].f >= 1 && J.j[k].f < width);
    J.start[k] = b;
    b += (J.j[k].n + 255) / 256;
  }
  J.start[J.n] = b;
  if (b == 0) return MPX_OK;
  CHECK_ARG(b < (1ll << 31));
  const u64 msk = ring_mask(width);
  cudaStream_t s = (cudaStream_t)stream;
  if (L <= 4)
    k_trunc_sub_multi<4><<<(unsigned)b, 256, 0, s>>>(J, L, msk, p0);
  else
    k_trunc_sub_multi<16><<<(unsigned)b, 256, 0, s>>>(J, L, msk, p0);
  return launch_status();
}

// Truncation fused with the layer plumbing around it (sim mode). The
// truncated tensor and its material order are the reference's; only where the
// result lands changes (derived.py:55-70 per element).
template <int LMAX>
__device__ __forceinline__ void trunc_elem(u64 (&out)[LMAX], const u64 (&xv)[LMAX], const u64* r_lo, i64 lo_ps,
                                           const u64* r_hi, i64 hi_ps, int L, i64 i, u64 msk, int f, u64 bias,
                                           u64 unbias, int p0) {
  u64 hv[LMAX];
  u64 s = 0;
#pragma unroll
  for (int l = 0; l < LMAX; ++l) {
    hv[l] = 0;
    if (l < L) {
      hv[l] = r_hi ? r_hi[l * hi_ps + i] : 0ull;
      u64 v = xv[l] + r_lo[l * lo_ps + i] + (hv[l] << f);
      if (l == p0) v += bias;
      s += v;
    }
  }
  const u64 chi = (s & msk) >> f;
#pragma unroll
  for (int l = 0; l < LMAX; ++l) {
    u64 v = 0ull - hv[l];
    if (l == p0) v += chi - unbias;
    out[l] = v & msk;
  }
}

// Conv output: z_nchw[l][b][c][s] = trunc(x[l][b*S+s][c] + (brow[l][c] << bshift)),
// 32 x 32 (s, c) tiles transposed through shared memory. nchw = 0 (linear
// layers): plain row order.
template <int LMAX>
__global__ void __launch_bounds__(256) k_trunc_rows_bias_nchw(u64* __restrict__ z, const u64* __restrict__ x,
                                                              const u64* __restrict__ brow, int bshift,
                                                              const u64* __restrict__ r_lo, i64 lo_ps,
                                                              const u64* __restrict__ r_hi, i64 hi_ps, int L,
                                                              i64 R, int S, int C, u64 msk, int f, u64 bias,
                                                              u64 unbias, int p0) {
  __shared__ u64 tile[LMAX][32][33];
  const i64 b = blockIdx.z;
  const int c0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const i64 n = R * C;
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    const int sl = ty + j, c = c0 + tx, sg = s0 + sl;
    if (c < C && sg < S) {
      const i64 i = (b * S + sg) * C + c;
      u64 xv[LMAX], o[LMAX];
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        xv[l] = l < L ? x[l * n + i] + (brow ? brow[l * C + c] << bshift : 0ull) : 0ull;
      trunc_elem<LMAX>(o, xv, r_lo, lo_ps, r_hi, hi_ps, L, i, msk, f, bias, unbias, p0);
#pragma unroll
      for (int l = 0; l < LMAX; ++l) tile[l][sl][tx] = o[l];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    const int cl = ty + j, c = c0 + cl, sg = s0 + tx;
    if (c < C && sg < S)
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) z[l * n + (b * C + c) * S + sg] = tile[l][tx][cl];
  }
}

template <int LMAX>
__global__ void k_trunc_rows_bias(u64* __restrict__ z, const u64* __restrict__ x, const u64* __restrict__ brow,
                                  int bshift, const u64* __restrict__ r_lo, i64 lo_ps, const u64* __restrict__ r_hi,
                                  i64 hi_ps, int L, i64 R, int C, u64 msk, int f, u64 bias, u64 unbias, int p0) {
  const i64 n = R * C;
  GRID_STRIDE(i, n) {
    const int c = (int)(i % C);
    u64 xv[LMAX], o[LMAX];
#pragma unroll
    for (int l = 0; l < LMAX; ++l)
      xv[l] = l < L ? x[l * n + i] + (brow ? brow[l * C + c] << bshift : 0ull) : 0ull;
    trunc_elem<LMAX>(o, xv, r_lo, lo_ps, r_hi, hi_ps, L, i, msk, f, bias, unbias, p0);
#pragma unroll
    for (int l = 0; l < LMAX; ++l)
      if (l < L) z[l * n + i] = o[l];
  }
}

extern "C" int mpx_trunc_rows_bias(uint64_t* z, const uint64_t* x, const uint64_t* brow, int bshift,
                                   const uint64_t* r_lo, int64_t lo_ps, const uint64_t* r_hi, int64_t hi_ps, int L,
                                   int64_t B, int64_t S, int64_t C, int nchw, int width, int f, uint64_t bias,
                                   uint64_t unbias, int p0, void* stream) {
  CHECK_ARG(z && x && r_lo && L >= 1 && L <= 8 && B >= 0 && S >= 1 && C >= 1 && width >= 2 && width <= 64 &&
            f >= 1 && f < width && bshift >= 0 && bshift < 64);
  const i64 R = B * S;
  if (R == 0) return MPX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const u64 msk = ring_mask(width);
  if (nchw) {
    CHECK_ARG(B <= 65535 && S < (1 << 30) && C < (1 << 30));
    dim3 grid((unsigned)((C + 31) / 32), (unsigned)((S + 31) / 32), (unsigned)B);
    CHECK_ARG(L <= 4);  // per-party 32 x 32 smem tiles
    k_trunc_rows_bias_nchw<4><<<grid, dim3(32, 8), 0, s>>>(z, x, brow, bshift, r_lo, lo_ps, r_hi, hi_ps, L, R,
                                                           (int)S, (int)C, msk, f, bias, unbias, p0);
  } else {
    CHECK_ARG(C < (1 << 30));
    if (L <= 4)
      k_trunc_rows_bias<4><<<grid_for(R * C), MPX_THREADS, 0, s>>>(z, x, brow, bshift, r_lo, lo_ps, r_hi, hi_ps,
                                                                   L, R, (int)C, msk, f, bias, unbias, p0);
    else
      k_trunc_rows_bias<8><<<grid_for(R * C), MPX_THREADS, 0, s>>>(z, x, brow, bshift, r_lo, lo_ps, r_hi, hi_ps,
                                                                   L, R, (int)C, msk, f, bias, unbias, p0);
  }
  return launch_status();
}

// Average-pool backward: d = trunc(dy) over dy's NCHW order, each value
// broadcast to its k x k window and stored in conv "rows" order
// z[l][(b*H + h)*W + w][c] (the layout the conv backward multiplies).
template <int LMAX>
__global__ void k_trunc_expand_rows(u64* __restrict__ z, const u64* __restrict__ x, const u64* __restrict__ r_lo,
                                    i64 lo_ps, const u64* __restrict__ r_hi, i64 hi_ps, int L, i64 B, int C, int Hs,
                                    int Ws, int k, u64 msk, int f, u64 bias, u64 unbias, int p0) {
  const i64 n = B * C * Hs * Ws;
  const i64 H = (i64)Hs * k, W = (i64)Ws * k;
  GRID_STRIDE(i, n) {
    const int ws = (int)(i % Ws);
    const i64 t1 = i / Ws;
    const int hs = (int)(t1 % Hs);
    const i64 t2 = t1 / Hs;
    const int c = (int)(t2 % C);
    const i64 b = t2 / C;
    u64 xv[LMAX], o[LMAX];
#pragma unroll
    for (int l = 0; l < LMAX; ++l) xv[l] = l < L ? x[l * n + i] : 0ull;
    trunc_elem<LMAX>(o, xv, r_lo, lo_ps, r_hi, hi_ps, L, i, msk, f, bias, unbias, p0);
    for (int a = 0; a < k; ++a)
      for (int bb = 0; bb < k; ++bb) {
        const i64 row = (b * H + (i64)hs * k + a) * W + (i64)ws * k + bb;
#pragma unroll
        for (int l = 0; l < LMAX; ++l)
          if (l < L) z[(i64)l * n * k * k + row * C + c] = o[l];
      }
  }
}

// Tiled variant: a CTA owns one (image b, source row hs): it truncates the
// row's C x Ws dy elements (all parties) into a shared tile, then writes the
// k output rows h = hs*k + a, all W = Ws*k columns and C channels in the
// output's own order (c fastest: coalesced stores, where the element-per-
// thread kernel above scatters 8-byte words C words apart).
template <int LMAX>
__global__ void __launch_bounds__(256) k_trunc_expand_rows_tiled(u64* __restrict__ z, const u64* __restrict__ x,
                                                                 const u64* __restrict__ r_lo, i64 lo_ps,
                                                                 const u64* __restrict__ r_hi, i64 hi_ps, int L,
                                                                 i64 B, int C, int Hs, int Ws, int k, u64 msk, int f,
                                                                 u64 bias, u64 unbias, int p0) {
  extern __shared__ u64 te_tile[];  // [LMAX][C][Ws]
  const i64 n = B * C * Hs * Ws;
  const int H = Hs * k, W = Ws * k;
  const i64 total = n * k * k;
  const int per = C * Ws;
  for (i64 bh = blockIdx.x; bh < B * Hs; bh += gridDim.x) {
    const i64 b = bh / Hs;
    const int hs = (int)(bh - b * Hs);
    for (int q = threadIdx.x; q < per; q += blockDim.x) {
      const int c = q / Ws, ws = q - c * Ws;
      const i64 i = ((b * C + c) * Hs + hs) * Ws + ws;
      u64 xv[LMAX], o[LMAX];
#pragma unroll
      for (int l = 0; l < LMAX; ++l) xv[l] = l < L ? __ldg(x + l * n + i) : 0ull;
      trunc_elem<LMAX>(o, xv, r_lo, lo_ps, r_hi, hi_ps, L, i, msk, f, bias, unbias, p0);
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) te_tile[(l * C + c) * Ws + ws] = o[l];
    }
    __syncthreads();
    const int outw = k * W * C;  // k output rows x W columns x C channels
    const i64 o0 = ((b * H + (i64)hs * k) * W) * C;
    for (int q = threadIdx.x; q < outw; q += blockDim.x) {
      const int c = q % C, rw = q / C;   // rw = a * W + w
      const int w = rw % W;
      const u64* tl = te_tile + c * Ws + w / k;
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) z[(i64)l * total + o0 + q] = tl[l * C * Ws];
    }
    __syncthreads();
  }
}

extern "C" int mpx_trunc_expand_rows(uint64_t* z, const uint64_t* x, const uint64_t* r_lo, int64_t lo_ps,
                                     const uint64_t* r_hi, int64_t hi_ps, int L, int64_t B, int64_t C, int64_t Hs,
                                     int64_t Ws, int64_t k, int width, int f, uint64_t bias, uint64_t unbias, int p0,
                                     void* stream) {
  CHECK_ARG(z && x && r_lo && L >= 1 && L <= 8 && B >= 0 && C >= 1 && Hs >= 1 && Ws >= 1 && k >= 1 &&
            C < (1 << 30) && Hs * k < (1 << 30) && Ws * k < (1 << 30) && width >= 2 && width <= 64 && f >= 1 &&
            f < width);
  const i64 n = B * C * Hs * Ws;
  if (n == 0) return MPX_OK;
  const size_t tsm = (size_t)4 * C * Ws * 8;
  if (L <= 4 && tsm <= 48 * 1024 && B * Hs < (1ll << 31)) {
    const unsigned g = (unsigned)min(B * Hs, (i64)dev_sms() * 8);
    k_trunc_expand_rows_tiled<4><<<g, 256, tsm, (cudaStream_t)stream>>>(
        z, x, r_lo, lo_ps, r_hi, hi_ps, L, B, (int)C, (int)Hs, (int)Ws, (int)k, ring_mask(width), f, bias, unbias, p0);
    return launch_status();
  }
  if (L <= 4)
    k_trunc_expand_rows<4><<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(
        z, x, r_lo, lo_ps, r_hi, hi_ps, L, B, (int)C, (int)Hs, (int)Ws, (int)k, ring_mask(width), f, bias, unbias, p0);
  else
    k_trunc_expand_rows<8><<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(
        z, x, r_lo, lo_ps, r_hi, hi_ps, L, B, (int)C, (int)Hs, (int)Ws, (int)k, ring_mask(width), f, bias, unbias, p0);
  return launch_status();
}

// ==========================================================================
// Binary Beaver AND on row-packed bits (basic.py:82-95)

__global__ void k_and_mask(u64* __restrict__ d, u64* __restrict__ e, const u64* __restrict__ x,
                           const u64* __restrict__ y, const u64* __restrict__ ta,
                           const u64* __restrict__ tb, i64 t_ps, i64 t_bit, int L, i64 rows, int m) {
  GRID_STRIDE(r, rows) {
    const i64 bit = t_bit + r * (i64)m;
    u64 dv = 0, ev = 0;
    for (int l = 0; l < L; ++l) {
      dv ^= x[l * rows + r] ^ load_bits(ta + l * t_ps, bit, m);
      ev ^= y[l * rows + r] ^ load_bits(tb + l * t_ps, bit, m);
    }
    const u64 mm = low_bits(m);
    d[r] = dv & mm;
    e[r] = ev & mm;
  }
}

__global__ void k_and_finish(u64* __restrict__ z, const u64* __restrict__ d, const u64* __restrict__ e,
                             const u64* __restrict__ ta, const u64* __restrict__ tb,
                             const u64* __restrict__ tc, i64 t_ps, i64 t_bit, int L, i64 rows, int m,
                             int p0) {
  const i64 total = (i64)L * rows;
  GRID_STRIDE(t, total) {
    const i64 l = L == 1 ? 0 : t / rows;
    const i64 r = t - l * rows;
    const i64 bit = t_bit + r * (i64)m;
    const u64 av = load_bits(ta + l * t_ps, bit, m);
    const u64 bv = load_bits(tb + l * t_ps, bit, m);
    const u64 cv = load_bits(tc + l * t_ps, bit, m);
    const u64 dv = d[r], ev = e[r];
    u64 v = cv ^ (dv & bv) ^ (ev & av);
    if (l == p0) v ^= dv & ev;
    z[t] = v & low_bits(m);
  }
}

extern "C" int mpx_and_mask(uint64_t* d, uint64_t* e, const uint64_t* x, const uint64_t* y,
                            const uint64_t* ta, const uint64_t* tb, int64_t t_ps, int64_t t_bit, int L,
                            int64_t rows, int m, void* stream) {
  CHECK_ARG(d && e && x && y && ta && tb && L >= 1 && rows >= 0 && m >= 1 && m <= 64 && t_bit >= 0);
  if (rows == 0) return MPX_OK;
  k_and_mask<<<grid_for(rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(d, e, x, y, ta, tb, t_ps, t_bit,
                                                                        L, rows, m);
  return launch_status();
}

extern "C" int mpx_and_finish(uint64_t* z, const uint64_t* d, const uint64_t* e, const uint64_t* ta,
                              const uint64_t* tb, const uint64_t* tc, int64_t t_ps, int64_t t_bit,
                              int L, int64_t rows, int m, int p0, void* stream) {
  CHECK_ARG(z && d && e && ta && tb && tc && L >= 1 && rows >= 0 && m >= 1 && m <= 64 && t_bit >= 0);
  if (rows == 0) return MPX_OK;
  k_and_finish<<<grid_for((i64)L * rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      z, d, e, ta, tb, tc, t_ps, t_bit, L, rows, m, p0);
  return launch_status();
}

// ==========================================================================
// Kogge-Stone carry level (basic.py:98-129). Positions j in [s, m) ("hi").
// Bintriple for the G-part bit j: t_bit + r*RW + (j - s); P-part:
// t_bit + r*RW + (m - s) + (j - s); RW = 2(m-s) (final level: m-s, G only).

struct CarryMat {
  u64 ag, bg, cg, ap, bp, cp;
};

__device__ __forceinline__ void carry_load(CarryMat& M, const u64* ta, const u64* tb, const u64* tc,
                                           i64 bit, int W, int s, bool last, bool need_c) {
  M.ag = load_bits(ta, bit, W) << s;
  M.bg = load_bits(tb, bit, W) << s;
  M.cg = need_c ? (load_bits(tc, bit, W) << s) : 0ull;
  if (!last) {
    M.ap = load_bits(ta, bit + W, W) << s;
    M.bp = load_bits(tb, bit + W, W) << s;
    M.cp = need_c ? (load_bits(tc, bit + W, W) << s) : 0ull;
  } else {
    M.ap = M.bp = M.cp = 0;
  }
}

__global__ void k_carry_mask(u64* __restrict__ dg, u64* __restrict__ eg, u64* __restrict__ dp,
                             u64* __restrict__ ep, const u64* __restrict__ G, const u64* __restrict__ P,
                             const u64* __restrict__ ta, const u64* __restrict__ tb, i64 t_ps,
                             i64 t_bit, int L, i64 rows, int m, int s, int last) {
  const int W = m - s;
  const int RW = last ? W : 2 * W;
  const u64 hi = low_bits(m) & ~low_bits(s);
  GRID_STRIDE(r, rows) {
    const i64 bit = t_bit + r * (i64)RW;
    u64 vdg = 0, veg = 0, vdp = 0, vep = 0;
    for (int l = 0; l < L; ++l) {
      CarryMat M;
      carry_load(M, ta + l * t_ps, tb + l * t_ps, nullptr, bit, W, s, last, false);
      const u64 g = G[l * rows + r], p = P[l * rows + r];
      const u64 left = p & hi;
      vdg ^= left ^ M.ag;
      veg ^= ((g << s) & hi) ^ M.bg;
      if (!last) {
        vdp ^= left ^ M.ap;
        vep ^= ((p << s) & hi) ^ M.bp;
      }
    }
    dg[r] = vdg;
    eg[r] = veg;
    if (!last) {
      dp[r] = vdp;
      ep[r] = vep;
    }
  }
}

__device__ __forceinline__ void carry_apply(u64& g, u64& p, const CarryMat& M, u64 vdg, u64 veg, u64 vdp,
                                            u64 vep, bool is_p0, bool last, int s) {
  u64 zg = M.cg ^ (vdg & M.bg) ^ (veg & M.ag);
  if (is_p0) zg ^= vdg & veg;
  g ^= zg;
  if (!last) {
    u64 zp = M.cp ^ (vdp & M.bp) ^ (vep & M.ap);
    if (is_p0) zp ^= vdp & vep;
    p = (p & low_bits(s)) | zp;
  }
}

__global__ void k_carry_finish(u64* __restrict__ G, u64* __restrict__ P, const u64* __restrict__ dg,
                               const u64* __restrict__ eg, const u64* __restrict__ dp,
                               const u64* __restrict__ ep, const u64* __restrict__ ta,
                               const u64* __restrict__ tb, const u64* __restrict__ tc, i64 t_ps,
                               i64 t_bit, int L, i64 rows, int m, int s, int last, int p0) {
  const int W = m - s;
  const int RW = last ? W : 2 * W;
  const i64 total = (i64)L * rows;
  GRID_STRIDE(t, total) {
    const i64 l = L == 1 ? 0 : t / rows;
    const i64 r = t - l * rows;
    CarryMat M;
    carry_load(M, ta + l * t_ps, tb + l * t_ps, tc + l * t_ps, t_bit + r * (i64)RW, W, s, last, true);
    u64 g = G[t], p = P[t];
    carry_apply(g, p, M, dg[r], eg[r], last ? 0 : dp[r], last ? 0 : ep[r], l == p0, last, s);
    G[t] = g;
    if (!last) P[t] = p;
  }
}

template <int LMAX>
__global__ void k_carry_fused(u64* __restrict__ G, u64* __restrict__ P, const u64* __restrict__ ta,
                              const u64* __restrict__ tb, const u64* __restrict__ tc, i64 t_ps,
                              i64 t_bit, int L, i64 rows, int m, int s, int last, int p0) {
  const int W = m - s;
  const int RW = last ? W : 2 * W;
  const u64 hi = low_bits(m) & ~low_bits(s);
  GRID_STRIDE(r, rows) {
    const i64 bit = t_bit + r * (i64)RW;
    CarryMat M[LMAX];
    u64 g[LMAX], p[LMAX];
    u64 vdg = 0, veg = 0, vdp = 0, vep = 0;
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        carry_load(M[l], ta + l * t_ps, tb + l * t_ps, tc + l * t_ps, bit, W, s, last, true);
        g[l] = G[l * rows + r];
        p[l] = P[l * rows + r];
        const u64 left = p[l] & hi;
        vdg ^= left ^ M[l].ag;
        veg ^= ((g[l] << s) & hi) ^ M[l].bg;
        vdp ^= left ^ M[l].ap;
        vep ^= ((p[l] << s) & hi) ^ M[l].bp;
      }
    }
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        carry_apply(g[l], p[l], M[l], vdg, veg, vdp, vep, l == p0, last, s);
        G[l * rows + r] = g[l];
        if (!last) P[l * rows + r] = p[l];
      }
    }
  }
}

extern "C" int mpx_carry_mask(uint64_t* dg, uint64_t* eg, uint64_t* dp, uint64_t* ep, const uint64_t* G,
                              const uint64_t* P, const uint64_t* ta, const uint64_t* tb, int64_t t_ps,
                              int64_t t_bit, int L, int64_t rows, int m, int s, int last, void* stream) {
  CHECK_ARG(dg && eg && G && P && ta && tb && L >= 1 && rows >= 0 && m >= 2 && m <= 64 && s >= 1 &&
            s < m && t_bit >= 0);
  CHECK_ARG(last || (dp && ep));
  if (rows == 0) return MPX_OK;
  k_carry_mask<<<grid_for(rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(dg, eg, dp, ep, G, P, ta, tb,
                                                                          t_ps, t_bit, L, rows, m, s,
                                                                          last);
  return launch_status();
}

extern "C" int mpx_carry_finish(uint64_t* G, uint64_t* P, const uint64_t* dg, const uint64_t* eg,
                                const uint64_t* dp, const uint64_t* ep, const uint64_t* ta,
                                const uint64_t* tb, const uint64_t* tc, int64_t t_ps, int64_t t_bit,
                                int L, int64_t rows, int m, int s, int last, int p0, void* stream) {
  CHECK_ARG(G && P && dg && eg && ta && tb && tc && L >= 1 && rows >= 0 && m >= 2 && m <= 64 &&
            s >= 1 && s < m && t_bit >= 0);
  CHECK_ARG(last || (dp && ep));
  if (rows == 0) return MPX_OK;
  k_carry_finish<<<grid_for((i64)L * rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      G, P, dg, eg, dp, ep, ta, tb, tc, t_ps, t_bit, L, rows, m, s, last, p0);
  return launch_status();
}

extern "C" int mpx_carry_fused(uint64_t* G, uint64_t* P, const uint64_t* ta, const uint64_t* tb,
                               const uint64_t* tc, int64_t t_ps, int64_t t_bit, int L, int64_t rows,
                               int m, int s, int last, int p0, void* stream) {
  CHECK_ARG(G && P && ta && tb && tc && L >= 1 && L <= 8 && rows >= 0 && m >= 2 && m <= 64 && s >= 1 &&
            s < m && t_bit >= 0);
  if (rows == 0) return MPX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (L <= 2)
    k_carry_fused<2><<<grid_for(rows), MPX_THREADS, 0, st>>>(G, P, ta, tb, tc, t_ps, t_bit, L, rows, m,
                                                             s, last, p0);
  else if (L <= 4)
    k_carry_fused<4><<<grid_for(rows), MPX_THREADS, 0, st>>>(G, P, ta, tb, tc, t_ps, t_bit, L, rows, m,
                                                             s, last, p0);
  else
    k_carry_fused<8><<<grid_for(rows), MPX_THREADS, 0, st>>>(G, P, ta, tb, tc, t_ps, t_bit, L, rows, m,
                                                             s, last, p0);
  return launch_status();
}

// G = x & pub ; P = P0 = x ^ [p0] pub   (basic.py:139-152)
__global__ void k_pubadd_init(u64* __restrict__ G, u64* __restrict__ P, u64* __restrict__ P0,
                              const u64* __restrict__ pub, const u64* __restrict__ x,
                              const u64* __restrict__ xb, i64 xb_ps, i64 xb_bit, int L, i64 rows, int m,
                              int p0) {
  const i64 total = (i64)L * rows;
  const u64 mm = low_bits(m);
  GRID_STRIDE(t, total) {
    const i64 l = L == 1 ? 0 : t / rows;
    const i64 r = t - l * rows;
    const u64 xv = x ? (x[t] & mm) : load_bits(xb + l * xb_ps, xb_bit + r * (i64)m, m);
    const u64 pv = pub[r] & mm;
    G[t] = xv & pv;
    const u64 p = (l == p0) ? (xv ^ pv) : xv;
    P[t] = p;
    P0[t] = p;
  }
}

extern "C" int mpx_pubadd_init(uint64_t* G, uint64_t* P, uint64_t* P0, const uint64_t* pub,
                               const uint64_t* x, const uint64_t* xb, int64_t xb_ps, int64_t xb_bit,
                               int L, int64_t rows, int m, int p0, void* stream) {
  CHECK_ARG(G && P && P0 && pub && (x || xb) && L >= 1 && rows >= 0 && m >= 1 && m <= 64 &&
            xb_bit >= 0);
  if (rows == 0) return MPX_OK;
  k_pubadd_init<<<grid_for((i64)L * rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      G, P, P0, pub, x, xb, xb_ps, xb_bit, L, rows, m, p0);
  return launch_status();
}

__global__ void k_sum_from_carries(u64* __restrict__ out, const u64* __restrict__ P0,
                                   const u64* __restrict__ G, i64 total, int m) {
  const u64 mm = low_bits(m);
  GRID_STRIDE(t, total) { out[t] = (P0[t] ^ (G[t] << 1)) & mm; }
}

extern "C" int mpx_sum_from_carries(uint64_t* out, const uint64_t* P0, const uint64_t* G, int L,
                                    int64_t rows, int m, void* stream) {
  CHECK_ARG(out && P0 && G && L >= 1 && rows >= 0 && m >= 1 && m <= 64);
  if (rows == 0) return MPX_OK;
  k_sum_from_carries<<<grid_for((i64)L * rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out, P0, G, (i64)L * rows, m);
  return launch_status();
}

// ==========================================================================
// Leftmost-one suffix OR (derived.py:131-149): lo = Y[:W], hi = Y[s:s+W],
// W = m - s; bintriple (r, j) = t_bit + r*W + j.

__global__ void k_lmo_mask(u64* __restrict__ d, u64* __restrict__ e, const u64* __restrict__ Y,
                           const u64* __restrict__ ta, const u64* __restrict__ tb, i64 t_ps, i64 t_bit,
                           int L, i64 rows, int m, int s) {
  const int W = m - s;
  const u64 mw = low_bits(W);
  GRID_STRIDE(r, rows) {
    const i64 bit = t_bit + r * (i64)W;
    u64 dv = 0, ev = 0;
    for (int l = 0; l < L; ++l) {
      const u64 y = Y[l * rows + r];
      dv ^= (y & mw) ^ load_bits(ta + l * t_ps, bit, W);
      ev ^= ((y >> s) & mw) ^ load_bits(tb + l * t_ps, bit, W);
    }
    d[r] = dv;
    e[r] = ev;
  }
}

__device__ __forceinline__ u64 lmo_apply(u64 y, u64 av, u64 bv, u64 cv, u64 dv, u64 ev, bool is_p0, int s,
                                         int W) {
  const u64 mw = low_bits(W);
  u64 z = cv ^ (dv & bv) ^ (ev & av);
  if (is_p0) z ^= dv & ev;
  const u64 lo = y & mw, hi = (y >> s) & mw;
  return (y & ~mw) | ((lo ^ hi ^ z) & mw);
}

__global__ void k_lmo_finish(u64* __restrict__ Y, const u64* __restrict__ d, const u64* __restrict__ e,
                             const u64* __restrict__ ta, const u64* __restrict__ tb,
                             const u64* __restrict__ tc, i64 t_ps, i64 t_bit, int L, i64 rows, int m,
                             int s, int p0) {
  const int W = m - s;
  const i64 total = (i64)L * rows;
  GRID_STRIDE(t, total) {
    const i64 l = L == 1 ? 0 : t / rows;
    const i64 r = t - l * rows;
    const i64 bit = t_bit + r * (i64)W;
    Y[t] = lmo_apply(Y[t], load_bits(ta + l * t_ps, bit, W), load_bits(tb + l * t_ps, bit, W),
                     load_bits(tc + l * t_ps, bit, W), d[r], e[r], l == p0, s, W);
  }
}

template <int LMAX>
__global__ void k_lmo_fused(u64* __restrict__ Y, const u64* __restrict__ ta, const u64* __restrict__ tb,
                            const u64* __restrict__ tc, i64 t_ps, i64 t_bit, int L, i64 rows, int m,
                            int s, int p0) {
  const int W = m - s;
  const u64 mw = low_bits(W);
  GRID_STRIDE(r, rows) {
    const i64 bit = t_bit + r * (i64)W;
    u64 y[LMAX], av[LMAX], bv[LMAX];
    u64 dv = 0, ev = 0;
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L) {
        y[l] = Y[l * rows + r];
        av[l] = load_bits(ta + l * t_ps, bit, W);
        bv[l] = load_bits(tb + l * t_ps, bit, W);
        dv ^= (y[l] & mw) ^ av[l];
        ev ^= ((y[l] >> s) & mw) ^ bv[l];
      }
    }
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l < L)
        Y[l * rows + r] =
            lmo_apply(y[l], av[l], bv[l], load_bits(tc + l * t_ps, bit, W), dv, ev, l == p0, s, W);
    }
  }
}

extern "C" int mpx_lmo_mask(uint64_t* d, uint64_t* e, const uint64_t* Y, const uint64_t* ta,
                            const uint64_t* tb, int64_t t_ps, int64_t t_bit, int L, int64_t rows, int m,
                            int s, void* stream) {
  CHECK_ARG(d && e && Y && ta && tb && L >= 1 && rows >= 0 && m >= 2 && m <= 64 && s >= 1 && s < m &&
            t_bit >= 0);
  if (rows == 0) return MPX_OK;
  k_lmo_mask<<<grid_for(rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(d, e, Y, ta, tb, t_ps, t_bit, L,
                                                                        rows, m, s);
  return launch_status();
}

extern "C" int mpx_lmo_finish(uint64_t* Y, const uint64_t* d, const uint64_t* e, const uint64_t* ta,
                              const uint64_t* tb, const uint64_t* tc, int64_t t_ps, int64_t t_bit, int L,
                              int64_t rows, int m, int s, int p0, void* stream) {
  CHECK_ARG(Y && d && e && ta && tb && tc && L >= 1 && rows >= 0 && m >= 2 && m <= 64 && s >= 1 &&
            s < m && t_bit >= 0);
  if (rows == 0) return MPX_OK;
  k_lmo_finish<<<grid_for((i64)L * rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      Y, d, e, ta, tb, tc, t_ps, t_bit, L, rows, m, s, p0);
  return launch_status();
}

extern "C" int mpx_lmo_fused(uint64_t* Y, const uint64_t* ta, const uint64_t* tb, const uint64_t* tc,
                             int64_t t_ps, int64_t t_bit, int L, int64_t rows, int m, int s, int p0,
                             void* stream) {
  CHECK_ARG(Y && ta && tb && tc && L >= 1 && L <= 8 && rows >= 0 && m >= 2 && m <= 64 && s >= 1 &&
            s < m && t_bit >= 0);
  if (rows == 0) return MPX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (L <= 2)
    k_lmo_fused<2><<<grid_for(rows), MPX_THREADS, 0, st>>>(Y, ta, tb, tc, t_ps, t_bit, L, rows, m, s, p0);
  else if (L <= 4)
    k_lmo_fused<4><<<grid_for(rows), MPX_THREADS, 0, st>>>(Y, ta, tb, tc, t_ps, t_bit, L, rows, m, s, p0);
  else
    k_lmo_fused<8><<<grid_for(rows), MPX_THREADS, 0, st>>>(Y, ta, tb, tc, t_ps, t_bit, L, rows, m, s, p0);
  return launch_status();
}

// ==========================================================================
// daBit conversion (basic.py:164-196)

__global__ void k_bit2a_mask(u64* __restrict__ c, const u64* __restrict__ b, const u64* __restrict__ rb,
                             i64 rb_ps, i64 rb_bit, int L, i64 rows, int m) {
  GRID_STRIDE(r, rows) {
    const i64 bit = rb_bit + r * (i64)m;
    u64 v = 0;
    for (int l = 0; l < L; ++l) v ^= b[l * rows + r] ^ load_bits(rb + l * rb_ps, bit, m);
    c[r] = v & low_bits(m);
  }
}

extern "C" int mpx_bit2a_mask(uint64_t* c, const uint64_t* b, const uint64_t* rbits, int64_t rb_ps,
                              int64_t rb_bit, int L, int64_t rows, int m, void* stream) {
  CHECK_ARG(c && b && rbits && L >= 1 && rows >= 0 && m >= 1 && m <= 64 && rb_bit >= 0);
  if (rows == 0) return MPX_OK;
  k_bit2a_mask<<<grid_for(rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(c, b, rbits, rb_ps, rb_bit, L,
                                                                          rows, m);
  return launch_status();
}

// mode 0: one thread per (l, r, j) output element, coalesced on r_arith.
__global__ void k_bit2a_expand(u64* __restrict__ out, const u64* __restrict__ c, const u64* __restrict__ ra,
                               i64 ra_ps, int L, i64 rows, int m, u64 msk, int p0) {
  const i64 per = rows * m;
  const i64 total = (i64)L * per;
  GRID_STRIDE(t, total) {
    const i64 l = L == 1 ? 0 : t / per;
    const i64 k = t - l * per;
    const i64 r = k / m;
    const int j = (int)(k - r * m);
    const u64 cj = (c[r] >> j) & 1ull;
    u64 v = ra[l * ra_ps + k] * (1ull - 2ull * cj);
    if (l == p0) v += cj;
    out[t] = v & msk;
  }
}

// mode 1 (compose): rows tiled through shared memory. A block stages the
// contiguous r_arith slab of B2A_ROWS rows (coalesced 16-byte loads), then 4
// threads per row reduce the weighted conversions with two shuffles.
#define B2A_ROWS 64
__global__ void __launch_bounds__(256) k_bit2a_compose(u64* __restrict__ out, const u64* __restrict__ c,
                                                       const u64* __restrict__ ra, i64 ra_ps, int L,
                                                       i64 rows, int m, u64 msk, int p0,
                                                       const u64* __restrict__ wts) {
  __shared__ __align__(16) u64 slab[B2A_ROWS * 64];
  __shared__ u64 wsh[64];
  if (threadIdx.x < 64) wsh[threadIdx.x] = wts ? (threadIdx.x < m ? wts[threadIdx.x] : 0ull)
                                               : (threadIdx.x < 64 ? (1ull << threadIdx.x) : 0ull);
  const i64 tiles = (rows + B2A_ROWS - 1) / B2A_ROWS;
  const i64 total = (i64)L * tiles;
  const int sub = threadIdx.x & 3;
  const int lr = threadIdx.x >> 2;  // local row 0..63
  for (i64 t = blockIdx.x; t < total; t += gridDim.x) {
    const i64 l = L == 1 ? 0 : t / tiles;
    const i64 r0 = (t - l * tiles) * B2A_ROWS;
    const int nr = (int)min((i64)B2A_ROWS, rows - r0);
    const u64* src = ra + l * ra_ps + r0 * (i64)m;
    const int nel = nr * m;
    __syncthreads();
    if ((((uintptr_t)src) & 15) == 0) {
      const int nv = nel >> 1;
      const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
      ulonglong2* d2 = reinterpret_cast<ulonglong2*>(slab);
      for (int i = threadIdx.x; i < nv; i += blockDim.x) d2[i] = __ldcs(s2 + i);
      if ((nel & 1) && threadIdx.x == 0) slab[nel - 1] = src[nel - 1];
    } else {
      for (int i = threadIdx.x; i < nel; i += blockDim.x) slab[i] = __ldcs(src + i);
    }
    __syncthreads();
    u64 acc = 0;
    if (lr < nr) {
      const u64 cw = c[r0 + lr];
      const u64* row = slab + lr * m;
      for (int j = sub; j < m; j += 4) {
        const u64 cj = (cw >> j) & 1ull;
        u64 v = row[j] * (1ull - 2ull * cj);
        if (l == p0) v += cj;
        acc += (v & msk) * wsh[j];
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (sub == 0 && lr < nr) out[l * rows + r0 + lr] = acc & msk;
  }
}

extern "C" int mpx_bit2a_finish(uint64_t* out, const uint64_t* c, const uint64_t* rarith, int64_t ra_ps,
                                int L, int64_t rows, int m, int width, int p0, const uint64_t* wts,
                                int mode, void* stream) {
  CHECK_ARG(out && c && rarith && L >= 1 && rows >= 0 && m >= 1 && m <= 64 && width >= 1 &&
            width <= 64 && (mode == 0 || mode == 1));
  if (rows == 0) return MPX_OK;
  const u64 msk = ring_mask(width);
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0)
    k_bit2a_expand<<<grid_for((i64)L * rows * m), MPX_THREADS, 0, s>>>(out, c, rarith, ra_ps, L, rows, m,
                                                                        msk, p0);
  else
  {
    i64 tiles = (i64)L * ((rows + B2A_ROWS - 1) / B2A_ROWS);
    unsigned g = (unsigned)(tiles < (i64)dev_sms() * 8 ? tiles : (i64)dev_sms() * 8);
    k_bit2a_compose<<<g, 256, 0, s>>>(out, c, rarith, ra_ps, L, rows, m, msk, p0, wts);
  }
  return launch_status();
}
