// Local ring arithmetic, codec, openings and bit-layout kernels.
//
// These are the HBM-bound elementwise pieces of the path (SURVEY §2.2 K3,
// K11, K12, K14): one pass, 64-bit words, grid-stride over all local
// parties. Reference: ring.py:20-134, sharing.py:37-121, session.py:71-115.
#include "common.cuh"

// --------------------------------------------------------------------------
// out = ka*a + kb*b + [l==p0](c0 + cv[i % cv_len])

__global__ void k_ring_lin(u64* __restrict__ out, const u64* __restrict__ a, u64 ka,
                           const u64* __restrict__ b, u64 kb, u64 c0, const u64* __restrict__ cv,
                           i64 cv_len, int L, i64 n, u64 msk, int p0) {
  // element-major with the party loop inside: no 64-bit division per word
  GRID_STRIDE(i, n) {
    for (int l = 0; l < L; ++l) {
      const i64 t = (i64)l * n + i;
      u64 v = a ? a[t] * ka : 0ull;
      if (b) v += b[t] * kb;
      if (l == p0) {
        v += c0;
        if (cv) v += cv[cv_len == n ? i : i % cv_len];
      }
      out[t] = v & msk;
    }
  }
}

extern "C" int mpx_ring_lin(uint64_t* out, const uint64_t* a, uint64_t ka, const uint64_t* b,
                            uint64_t kb, uint64_t c0, const uint64_t* cv, int64_t cv_len, int L,
                            int64_t n, int width, int p0, void* stream) {
  CHECK_ARG(out && L >= 1 && n >= 0 && width >= 1 && width <= 64);
  CHECK_ARG(!cv || cv_len >= 1);
  if (n == 0) return MPX_OK;
  k_ring_lin<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(
      out, a, ka, b, kb, c0, cv, cv_len, L, n, ring_mask(width), p0);
  return launch_status();
}

__global__ void k_ring_mul(u64* __restrict__ out, const u64* __restrict__ a, const u64* __restrict__ b,
                           i64 n, u64 msk) {
  GRID_STRIDE(i, n) { out[i] = (a[i] * b[i]) & msk; }
}

extern "C" int mpx_ring_mul(uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, int width,
                            void* stream) {
  CHECK_ARG(out && a && b && n >= 0 && width >= 1 && width <= 64);
  if (n == 0) return MPX_OK;
  k_ring_mul<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, a, b, n, ring_mask(width));
  return launch_status();
}

// --------------------------------------------------------------------------
// Row dot with public weights: one warp per row, lanes stride the row
// (coalesced), u64 shuffle reduction. K12 (row sums) and compose contractions.

__global__ void k_ring_rowdot(u64* __restrict__ out, const u64* __restrict__ x,
                              const u64* __restrict__ wts, i64 nrows, i64 cols, u64 msk) {
  const int lane = threadIdx.x & 31;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 r = warp; r < nrows; r += nwarps) {
    const u64* row = x + r * cols;
    u64 acc = 0;
    for (i64 j = lane; j < cols; j += 32) acc += wts ? row[j] * wts[j] : row[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = acc & msk;
  }
}

// Short rows: one thread per row (cols <= 8 keeps the loads in a few sectors).
__global__ void k_ring_rowdot_small(u64* __restrict__ out, const u64* __restrict__ x,
                                    const u64* __restrict__ wts, i64 nrows, i64 cols, u64 msk) {
  GRID_STRIDE(r, nrows) {
    const u64* row = x + r * cols;
    u64 acc = 0;
    for (i64 j = 0; j < cols; ++j) acc += wts ? row[j] * wts[j] : row[j];
    out[r] = acc & msk;
  }
}

extern "C" int mpx_ring_rowdot(uint64_t* out, const uint64_t* x, const uint64_t* wts, int L,
                               int64_t rows, int64_t cols, int width, void* stream) {
  CHECK_ARG(out && x && L >= 1 && rows >= 0 && cols >= 1 && width >= 1 && width <= 64);
  const i64 nrows = (i64)L * rows;
  if (nrows == 0) return MPX_OK;
  if (cols <= 8)
    k_ring_rowdot_small<<<grid_for(nrows), MPX_THREADS, 0, (cudaStream_t)stream>>>(
        out, x, wts, nrows, cols, ring_mask(width));
  else
    k_ring_rowdot<<<grid_for(nrows * 32), MPX_THREADS, 0, (cudaStream_t)stream>>>(
        out, x, wts, nrows, cols, ring_mask(width));
  return launch_status();
}

// Column sums of [L][rows][cols] -> [L][cols] (the bias gradient: a sum over
// the batch / spatial rows). Narrow tables (cols <= blockDim) tile a block as
// (blockDim / cols) row lanes x cols, so consecutive threads read consecutive
// words; partial sums meet in shared memory, then one wrapping atomic per
// column and block. Wide tables walk columns directly.
__global__ void k_ring_colsum(u64* __restrict__ out, const u64* __restrict__ x, i64 rows, int cols,
                              i64 rows_per_block) {
  extern __shared__ u64 part[];
  const int l = blockIdx.y;
  x += (i64)l * rows * cols;
  out += (i64)l * cols;
  const i64 r0 = (i64)blockIdx.x * rows_per_block;
  const i64 r1 = min(rows, r0 + rows_per_block);
  if (cols <= (int)blockDim.x) {
    const int lanes = blockDim.x / cols;
    const int col = threadIdx.x % cols, sub = threadIdx.x / cols;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) part[c] = 0;
    __syncthreads();
    if (sub < lanes) {
      u64 acc = 0;
      for (i64 r = r0 + sub; r < r1; r += lanes) acc += x[r * cols + col];
      atomicAdd(reinterpret_cast<unsigned long long*>(&part[col]), (unsigned long long)acc);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cols; c += blockDim.x)
      atomicAdd(reinterpret_cast<unsigned long long*>(&out[c]), (unsigned long long)part[c]);
  } else {
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      u64 acc = 0;
      for (i64 r = r0; r < r1; ++r) acc += x[r * cols + c];
      atomicAdd(reinterpret_cast<unsigned long long*>(&out[c]), (unsigned long long)acc);
    }
  }
}

__global__ void k_mask_inplace(u64* __restrict__ v, i64 n, u64 msk) {
  GRID_STRIDE(i, n) v[i] &= msk;
}

extern "C" int mpx_ring_colsum(uint64_t* out, const uint64_t* x, int L, int64_t rows, int64_t cols, int width,
                               void* stream) {
  CHECK_ARG(out && x && L >= 1 && L <= 65535 && rows >= 0 && cols >= 1 && cols <= (1 << 20) && width >= 1 &&
            width <= 64);
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(out, 0, (size_t)L * cols * 8, s) != cudaSuccess) return MPX_ERR_CUDA;
  if (rows == 0) return MPX_OK;
  const int threads = 256;
  // enough blocks to cover the SMs a few times, each a contiguous row band
  const i64 lanes = cols <= threads ? threads / cols : 1;
  i64 nblk = (4 * (i64)dev_sms() + L - 1) / L;
  const i64 min_rows = 4 * lanes;
  nblk = max((i64)1, min(nblk, (rows + min_rows - 1) / min_rows));
  const i64 rpb = (rows + nblk - 1) / nblk;
  nblk = (rows + rpb - 1) / rpb;
  const size_t sm = cols <= threads ? (size_t)cols * 8 : 0;
  k_ring_colsum<<<dim3((unsigned)nblk, (unsigned)L), threads, sm, s>>>(out, x, rows, (int)cols, rpb);
  if (width < 64) k_mask_inplace<<<grid_for((i64)L * cols), MPX_THREADS, 0, s>>>(out, (i64)L * cols, ring_mask(width));
  return launch_status();
}

// z[l][r][c] += b[l][c] << shift (a bias row lifted to the product's
// precision and broadcast over rows), in place.
__global__ void k_ring_add_rowvec(u64* __restrict__ z, const u64* __restrict__ b, i64 rows, int cols, int shift,
                                  u64 msk, i64 total) {
  GRID_STRIDE(t, total) {
    const i64 c = t % cols;
    const i64 l = t / ((i64)rows * cols);
    z[t] = (z[t] + (b[l * cols + c] << shift)) & msk;
  }
}

extern "C" int mpx_ring_add_rowvec(uint64_t* z, const uint64_t* b, int L, int64_t rows, int64_t cols, int shift,
                                   int width, void* stream) {
  CHECK_ARG(z && b && L >= 1 && rows >= 0 && cols >= 1 && shift >= 0 && shift < 64 && width >= 1 && width <= 64);
  const i64 total = (i64)L * rows * cols;
  if (total == 0) return MPX_OK;
  k_ring_add_rowvec<<<grid_for(total), MPX_THREADS, 0, (cudaStream_t)stream>>>(z, b, rows, (int)cols, shift,
                                                                                ring_mask(width), total);
  return launch_status();
}

// k x k window sums with stride st over [planes][H][W] -> [planes][OH][OW],
// OH = (H - k) / st + 1 (average pooling before its scaling).
__global__ void k_ring_pool_sum(u64* __restrict__ out, const u64* __restrict__ x, i64 planes, int H, int W,
                                int k, int st, int OH, int OW, u64 msk) {
  const i64 n = planes * OH * OW;
  GRID_STRIDE(i, n) {
    const int oj = (int)(i % OW);
    const i64 t = i / OW;
    const int oi = (int)(t % OH);
    const i64 p = t / OH;
    const u64* src = x + (p * H + (i64)oi * st) * W + (i64)oj * st;
    u64 acc = 0;
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) acc += src[(i64)a * W + b];
    out[i] = acc & msk;
  }
}

extern "C" int mpx_ring_pool_sum(uint64_t* out, const uint64_t* x, int64_t planes, int64_t H, int64_t W,
                                 int64_t k, int64_t stride, int width, void* stream) {
  CHECK_ARG(out && x && planes >= 0 && k >= 1 && stride >= 1 && H >= k && W >= k && H < (1 << 20) &&
            W < (1 << 20) && width >= 1 && width <= 64);
  const int OH = (int)((H - k) / stride + 1), OW = (int)((W - k) / stride + 1);
  const i64 n = planes * OH * OW;
  if (n == 0) return MPX_OK;
  k_ring_pool_sum<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, x, planes, (int)H, (int)W, (int)k,
                                                                          (int)stride, OH, OW, ring_mask(width));
  return launch_status();
}

// Adjoint of the window sum: dx[p][h][w] = sum of d over the windows that
// cover (h, w) (average-pool backward, overlapping windows allowed).
__global__ void k_ring_pool_scatter(u64* __restrict__ dx, const u64* __restrict__ d, i64 planes, int H, int W,
                                    int k, int st, int OH, int OW, u64 msk) {
  const i64 n = planes * H * W;
  GRID_STRIDE(i, n) {
    const int w = (int)(i % W);
    const i64 t = i / W;
    const int h = (int)(t % H);
    const i64 p = t / H;
    // windows oi with oi*st <= h < oi*st + k
    const int oi_hi = min(OH - 1, h / st), oj_hi = min(OW - 1, w / st);
    const int oi_lo = max(0, (h - k + st) / st), oj_lo = max(0, (w - k + st) / st);
    u64 acc = 0;
    for (int oi = oi_lo; oi <= oi_hi; ++oi) {
      if (h >= oi * st + k) continue;
      for (int oj = oj_lo; oj <= oj_hi; ++oj) {
        if (w >= oj * st + k) continue;
        acc += d[(p * OH + oi) * OW + oj];
      }
    }
    dx[i] = acc & msk;
  }
}

extern "C" int mpx_ring_pool_scatter(uint64_t* dx, const uint64_t* d, int64_t planes, int64_t H, int64_t W,
                                     int64_t k, int64_t stride, int width, void* stream) {
  CHECK_ARG(dx && d && planes >= 0 && k >= 1 && stride >= 1 && H >= k && W >= k && H < (1 << 20) &&
            W < (1 << 20) && width >= 1 && width <= 64);
  const int OH = (int)((H - k) / stride + 1), OW = (int)((W - k) / stride + 1);
  const i64 n = planes * H * W;
  if (n == 0) return MPX_OK;
  k_ring_pool_scatter<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(dx, d, planes, (int)H, (int)W, (int)k,
                                                                              (int)stride, OH, OW, ring_mask(width));
  return launch_status();
}

// --------------------------------------------------------------------------
// Codec: floor(x * 2^f) as int64, two's complement into Z_2^w (ring.py:76-89)

__global__ void k_encode(u64* __restrict__ out, const double* __restrict__ in, i64 n, double scale,
                         u64 msk) {
  GRID_STRIDE(i, n) {
    const double s = floor(in[i] * scale);
    // numpy's float64 -> int64 cast on x86 (cvttsd2si) yields INT64_MIN for
    // NaN and for anything outside [-2^63, 2^63); CUDA's cvt saturates, so
    // the reference's out-of-range encodings are reproduced explicitly.
    const bool in_range = s >= -9223372036854775808.0 && s < 9223372036854775808.0;
    out[i] = (in_range ? (u64)(long long)s : 0x8000000000000000ull) & msk;
  }
}

// Centered representative in [-2^(w-1), 2^(w-1)) as int64 (ring.py:65-73).
__global__ void k_to_signed(long long* __restrict__ out, const u64* __restrict__ in, i64 n, int w) {
  GRID_STRIDE(i, n) {
    const u64 v = in[i] & ring_mask(w);
    out[i] = (w == 64 || !(v >> (w - 1))) ? (long long)v : (long long)(v | ~ring_mask(w));
  }
}

__global__ void k_decode(double* __restrict__ out, const u64* __restrict__ in, i64 n, int w,
                         double inv_scale) {
  GRID_STRIDE(i, n) {
    u64 v = in[i] & ring_mask(w);
    long long s;
    if (w == 64) {
      s = (long long)v;
    } else {
      const u64 sign = 1ull << (w - 1);
      s = (v & sign) ? (long long)(v | ~ring_mask(w)) : (long long)v;
    }
    out[i] = (double)s * inv_scale;
  }
}

extern "C" int mpx_encode(uint64_t* out, const double* in, int64_t n, int width, int frac,
                          void* stream) {
  CHECK_ARG(out && in && n >= 0 && width >= 1 && width <= 64 && frac >= 0 && frac < 64);
  if (n == 0) return MPX_OK;
  k_encode<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, in, n, ldexp(1.0, frac),
                                                                   ring_mask(width));
  return launch_status();
}

extern "C" int mpx_to_signed(int64_t* out, const uint64_t* in, int64_t n, int width, void* stream) {
  CHECK_ARG(out && in && n >= 0 && width >= 1 && width <= 64);
  if (n == 0) return MPX_OK;
  k_to_signed<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>((long long*)out, in, n, width);
  return launch_status();
}

extern "C" int mpx_decode(double* out, const uint64_t* in, int64_t n, int width, int frac,
                          void* stream) {
  CHECK_ARG(out && in && n >= 0 && width >= 1 && width <= 64 && frac >= 0 && frac < 64);
  if (n == 0) return MPX_OK;
  k_decode<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, in, n, width,
                                                                   ldexp(1.0, -frac));
  return launch_status();
}

// --------------------------------------------------------------------------
// Openings (session.py:87-115): reduce the local parties' contributions.

__global__ void k_open_sum(u64* __restrict__ out, const u64* __restrict__ x, int L, i64 n, u64 msk) {
  GRID_STRIDE(i, n) {
    u64 s = 0;
    for (int l = 0; l < L; ++l) s += x[(i64)l * n + i];
    out[i] = s & msk;
  }
}

__global__ void k_open_xor(u64* __restrict__ out, const u64* __restrict__ x, int L, i64 n) {
  GRID_STRIDE(i, n) {
    u64 s = 0;
    for (int l = 0; l < L; ++l) s ^= x[(i64)l * n + i];
    out[i] = s;
  }
}

__global__ void k_mask_sub(u64* __restrict__ out, const u64* __restrict__ x, const u64* __restrict__ a,
                           i64 a_ps, int L, i64 n, u64 msk) {
  GRID_STRIDE(i, n) {
    u64 s = 0;
    for (int l = 0; l < L; ++l) s += x[(i64)l * n + i] - a[(i64)l * a_ps + i];
    out[i] = s & msk;
  }
}

extern "C" int mpx_open_sum(uint64_t* out, const uint64_t* x, int L, int64_t n, int width,
                            void* stream) {
  CHECK_ARG(out && x && L >= 1 && n >= 0 && width >= 1 && width <= 64);
  if (n == 0) return MPX_OK;
  k_open_sum<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, x, L, n, ring_mask(width));
  return launch_status();
}

extern "C" int mpx_open_xor(uint64_t* out, const uint64_t* x, int L, int64_t n, void* stream) {
  CHECK_ARG(out && x && L >= 1 && n >= 0);
  if (n == 0) return MPX_OK;
  k_open_xor<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, x, L, n);
  return launch_status();
}

extern "C" int mpx_mask_sub(uint64_t* out, const uint64_t* x, const uint64_t* a, int64_t a_ps, int L,
                            int64_t n, int width, void* stream) {
  CHECK_ARG(out && x && a && L >= 1 && n >= 0 && width >= 1 && width <= 64);
  if (n == 0) return MPX_OK;
  k_mask_sub<<<grid_for(n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, x, a, a_ps, L, n,
                                                                     ring_mask(width));
  return launch_status();
}

// Beaver masks of a batch of operands read in place (one launch for all the
// equal-shape products of a batch_matmul round):
//   out[b][j] = sum_l (x_l[b][j] - a_l[b][j]) mod 2^w,
// x at party stride x_ps and batch stride x_bs, a at a_ps / a_bs.
__global__ void k_mask_sub_bs(u64* __restrict__ out, const u64* __restrict__ x, i64 x_ps, i64 x_bs,
                              const u64* __restrict__ a, i64 a_ps, i64 a_bs, int L, i64 batch, i64 n, u64 msk) {
  const i64 total = batch * n;
  GRID_STRIDE(t, total) {
    const i64 b = t / n, j = t - b * n;
    u64 s = 0;
    for (int l = 0; l < L; ++l) s += x[(i64)l * x_ps + b * x_bs + j] - a[(i64)l * a_ps + b * a_bs + j];
    out[t] = s & msk;
  }
}

extern "C" int mpx_mask_sub_bs(uint64_t* out, const uint64_t* x, int64_t x_ps, int64_t x_bs, const uint64_t* a,
                               int64_t a_ps, int64_t a_bs, int L, int64_t batch, int64_t n, int width,
                               void* stream) {
  CHECK_ARG(out && x && a && L >= 1 && batch >= 0 && n >= 0 && width >= 1 && width <= 64);
  if (batch == 0 || n == 0) return MPX_OK;
  k_mask_sub_bs<<<grid_for(batch * n), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, x, x_ps, x_bs, a, a_ps, a_bs,
                                                                              L, batch, n, ring_mask(width));
  return launch_status();
}

// Same for transposed operands without materialising the transpose:
// out[b][r][c] = sum_l (x_l[b][c][r] - a_l[b][r][c]) mod 2^w, x_l[b] stored
// cols x rows. 32 x 32 tiles through shared memory: x is read along its rows,
// a and out along theirs.
__global__ void k_mask_sub_t(u64* __restrict__ out, const u64* __restrict__ x, i64 x_ps, i64 x_bs,
                             const u64* __restrict__ a, i64 a_ps, i64 a_bs, int L, i64 rows, i64 cols, u64 msk) {
  __shared__ u64 tile[32][33];
  const i64 bt = blockIdx.z;
  x += bt * x_bs;
  a += bt * a_bs;
  out += bt * rows * cols;
  const i64 r0 = (i64)blockIdx.y * 32, c0 = (i64)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    const i64 c = c0 + ty + j, r = r0 + tx;
    u64 s = 0;
    if (c < cols && r < rows)
      for (int l = 0; l < L; ++l) s += x[(i64)l * x_ps + c * rows + r];
    tile[ty + j][tx] = s;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    const i64 r = r0 + ty + j, c = c0 + tx;
    if (r < rows && c < cols) {
      u64 s = tile[tx][ty + j];
      for (int l = 0; l < L; ++l) s -= a[(i64)l * a_ps + r * cols + c];
      out[r * cols + c] = s & msk;
    }
  }
}

extern "C" int mpx_mask_sub_t(uint64_t* out, const uint64_t* x, int64_t x_ps, int64_t x_bs, const uint64_t* a,
                              int64_t a_ps, int64_t a_bs, int L, int64_t batch, int64_t rows, int64_t cols,
                              int width, void* stream) {
  CHECK_ARG(out && x && a && L >= 1 && batch >= 0 && rows >= 0 && cols >= 0 && width >= 1 && width <= 64);
  if (batch == 0 || rows == 0 || cols == 0) return MPX_OK;
  CHECK_ARG((rows + 31) / 32 <= 65535 && batch <= 65535);
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32), (unsigned)batch);
  k_mask_sub_t<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(out, x, x_ps, x_bs, a, a_ps, a_bs, L, rows, cols,
                                                                ring_mask(width));
  return launch_status();
}

// --------------------------------------------------------------------------
// Local bit ops on row-packed words.

__global__ void k_bits_op(u64* __restrict__ out, const u64* __restrict__ a, const u64* __restrict__ b,
                          int op, int L, i64 rows, int m, int p0, int imm) {
  const i64 total = (i64)L * rows;
  const u64 mm = low_bits(m);
  GRID_STRIDE(t, total) {
    const i64 l = L == 1 ? 0 : t / rows;
    const i64 r = t - l * rows;
    const u64 x = a[t];
    u64 v;
    switch (op) {
      case MPX_BITS_XOR: v = x ^ b[t]; break;
      case MPX_BITS_AND: v = x & b[t]; break;
      case MPX_BITS_AND_PUB: v = x & b[r]; break;
      case MPX_BITS_XOR_PUB: v = (l == p0) ? (x ^ b[r]) : x; break;
      case MPX_BITS_XOR_SHR1: v = x ^ ((x & mm) >> 1); break;
      case MPX_BITS_PARITY: v = (u64)(__popcll(x & mm) & 1); break;
      case MPX_BITS_SIGNFOLD: v = (x & mm) ^ (((x >> m) & 1ull) ? mm : 0ull); break;
      case MPX_BITS_SHL_OR: v = (x & low_bits(imm)) | (b[t] << imm); break;
      case MPX_BITS_BCAST_PUB: v = (l == p0) ? (x ^ b[0]) : x; break;
      default: v = 0; break;
    }
    out[t] = (op == MPX_BITS_SIGNFOLD || op == MPX_BITS_PARITY) ? v : (v & mm);
  }
}

extern "C" int mpx_bits_op(uint64_t* out, const uint64_t* a, const uint64_t* b, int op, int L,
                           int64_t rows, int m, int p0, int imm, void* stream) {
  CHECK_ARG(out && a && L >= 1 && rows >= 0 && m >= 1 && m <= 64 && op >= 0 && op <= 8);
  CHECK_ARG(b || op == MPX_BITS_XOR_SHR1 || op == MPX_BITS_PARITY || op == MPX_BITS_SIGNFOLD);
  CHECK_ARG(op != MPX_BITS_SIGNFOLD || m < 64);
  CHECK_ARG(op != MPX_BITS_SHL_OR || (imm >= 0 && imm < 64));
  if (rows == 0) return MPX_OK;
  k_bits_op<<<grid_for((i64)L * rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, a, b, op, L, rows,
                                                                                m, p0, imm);
  return launch_status();
}

struct GatherSpec {
  int8_t src[64];
};

// General bit gather (arbitrary source list).
__global__ void k_bits_gather(u64* __restrict__ out, const u64* __restrict__ in, GatherSpec g, int k,
                              i64 n) {
  GRID_STRIDE(i, n) {
    const u64 x = in[i];
    u64 v = 0;
#pragma unroll 8
    for (int t = 0; t < k; ++t) {
      const int s = g.src[t];
      if (s >= 0) v |= ((x >> s) & 1ull) << t;
    }
    out[i] = v;
  }
}

// Fast paths: up to 3 runs, each a contiguous ascending (shift + mask) or
// descending (bit reverse) source range; -1 padding runs produce zeros.
struct RunSpec {
  int nruns;
  int src0[3], len[3], dst0[3], dir[3];  // dir: +1 ascending, -1 descending, 0 zeros
};

__global__ void k_bits_runs(u64* __restrict__ out, const u64* __restrict__ in, RunSpec rs, i64 n) {
  GRID_STRIDE(i, n) {
    const u64 x = in[i];
    u64 v = 0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q >= rs.nruns) break;
      const int len = rs.len[q];
      if (rs.dir[q] > 0) {
        v |= ((x >> rs.src0[q]) & low_bits(len)) << rs.dst0[q];
      } else if (rs.dir[q] < 0) {
        // bits src0, src0-1, ..., src0-len+1 -> dst0, dst0+1, ...
        const u64 seg = (x >> (rs.src0[q] - len + 1)) & low_bits(len);
        v |= (__brevll(seg) >> (64 - len)) << rs.dst0[q];
      }
    }
    out[i] = v;
  }
}

static bool make_runs(const GatherSpec& g, int k, RunSpec& rs) {
  rs.nruns = 0;
  int t = 0;
  while (t < k) {
    if (rs.nruns == 3) return false;
    const int q = rs.nruns++;
    rs.dst0[q] = t;
    rs.src0[q] = g.src[t];
    if (g.src[t] < 0) {
      int e = t;
      while (e < k && g.src[e] < 0) ++e;
      rs.len[q] = e - t;
      rs.dir[q] = 0;
      t = e;
      continue;
    }
    int e = t + 1;
    int dir = 0;
    if (e < k && g.src[e] == g.src[t] + 1) dir = 1;
    else if (e < k && g.src[e] == g.src[t] - 1) dir = -1;
    else dir = 1;
    while (e < k && g.src[e] >= 0 && g.src[e] == g.src[e - 1] + dir) ++e;
    rs.len[q] = e - t;
    rs.dir[q] = dir;
    t = e;
  }
  return true;
}

extern "C" int mpx_bits_gather(uint64_t* out, const uint64_t* in, const int8_t* src_host, int k,
                               int64_t nwords, void* stream) {
  CHECK_ARG(out && in && src_host && k >= 1 && k <= 64 && nwords >= 0);
  GatherSpec g;
  for (int t = 0; t < 64; ++t) g.src[t] = t < k ? src_host[t] : (int8_t)-1;
  for (int t = 0; t < k; ++t) CHECK_ARG(g.src[t] < 64);
  if (nwords == 0) return MPX_OK;
  RunSpec rs;
  if (make_runs(g, k, rs))
    k_bits_runs<<<grid_for(nwords), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, in, rs, nwords);
  else
    k_bits_gather<<<grid_for(nwords), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, in, g, k, nwords);
  return launch_status();
}

__global__ void k_bits_pack(u64* __restrict__ out, const uint8_t* __restrict__ in, i64 rows, int m) {
  GRID_STRIDE(r, rows) {
    const uint8_t* row = in + r * m;
    u64 v = 0;
    for (int j = 0; j < m; ++j) v |= (u64)(row[j] & 1u) << j;
    out[r] = v;
  }
}

__global__ void k_bits_unpack(uint8_t* __restrict__ out, const u64* __restrict__ in, i64 rows, int m) {
  const i64 total = rows * m;
  GRID_STRIDE(t, total) {
    const i64 r = t / m;
    const int j = (int)(t - r * m);
    out[t] = (uint8_t)((in[r] >> j) & 1ull);
  }
}

extern "C" int mpx_bits_pack(uint64_t* out, const uint8_t* in, int64_t rows, int m, void* stream) {
  CHECK_ARG(out && in && rows >= 0 && m >= 1 && m <= 64);
  if (rows == 0) return MPX_OK;
  k_bits_pack<<<grid_for(rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, in, rows, m);
  return launch_status();
}

extern "C" int mpx_bits_unpack(uint8_t* out, const uint64_t* in, int64_t rows, int m, void* stream) {
  CHECK_ARG(out && in && rows >= 0 && m >= 1 && m <= 64);
  if (rows == 0) return MPX_OK;
  k_bits_unpack<<<grid_for(rows * m), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, in, rows, m);
  return launch_status();
}

__global__ void k_bits_flat_to_rows(u64* __restrict__ out, const u64* __restrict__ flat, i64 flat_bit,
                                    i64 rows, int m) {
  GRID_STRIDE(r, rows) { out[r] = load_bits(flat, flat_bit + r * (i64)m, m); }
}

// One thread per output word of the flat stream: bit t = row t/m, bit t%m.
__global__ void k_bits_rows_to_flat(u64* __restrict__ flat, const u64* __restrict__ rin, i64 rows,
                                    int m) {
  const i64 nbits = rows * m;
  const i64 nw = (nbits + 63) >> 6;
  GRID_STRIDE(w, nw) {
    u64 v = 0;
    const i64 t0 = w << 6;
    i64 r = t0 / m;
    int j = (int)(t0 - r * m);
    for (int b = 0; b < 64 && t0 + b < nbits; ++b) {
      v |= ((rin[r] >> j) & 1ull) << b;
      if (++j == m) {
        j = 0;
        ++r;
      }
    }
    flat[w] = v;
  }
}

extern "C" int mpx_bits_flat_to_rows(uint64_t* out, const uint64_t* flat, int64_t flat_bit,
                                     int64_t rows, int m, void* stream) {
  CHECK_ARG(out && flat && flat_bit >= 0 && rows >= 0 && m >= 1 && m <= 64);
  if (rows == 0) return MPX_OK;
  k_bits_flat_to_rows<<<grid_for(rows), MPX_THREADS, 0, (cudaStream_t)stream>>>(out, flat, flat_bit,
                                                                                 rows, m);
  return launch_status();
}

extern "C" int mpx_bits_rows_to_flat(uint64_t* flat, const uint64_t* rows_in, int64_t rows, int m,
                                     void* stream) {
  CHECK_ARG(flat && rows_in && rows >= 0 && m >= 1 && m <= 64);
  if (rows == 0) return MPX_OK;
  const i64 nw = (rows * m + 63) >> 6;
  k_bits_rows_to_flat<<<grid_for(nw), MPX_THREADS, 0, (cudaStream_t)stream>>>(flat, rows_in, rows, m);
  return launch_status();
}

// --------------------------------------------------------------------------
// Diagnostics

extern "C" const char* mpx_version(void) { return "libmpx 0.1 sm_100a"; }

extern "C" int mpx_last_cuda_error(void) { return (int)cudaGetLastError(); }

extern "C" const char* mpx_cuda_error_string(int code) {
  return cudaGetErrorString((cudaError_t)code);
}

extern "C" int mpx_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

// --------------------------------------------------------------------------
// Convolution layout ops on shares (local, linear): im2col gathers, col2im
// scatter-adds mod 2^w. x: [L][B][C][H][W]; cols: [L][B*OH*OW][C*K*K].

// Index math in IT (u32 whenever the tensor fits: 64-bit division costs
// ~10x more and dominated these gathers).
template <typename IT>
__global__ void k_im2col(u64* __restrict__ out, const u64* __restrict__ x, IT B, IT C, IT H, IT W, IT K, IT S,
                         IT P, IT OH, IT OW, IT total) {
  const IT cols = C * K * K;
  const IT rows = B * OH * OW;
  for (IT t = (IT)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (IT)gridDim.x * blockDim.x) {
    const IT col = t % cols;
    const IT rr = t / cols;
    const IT row = rr % rows;
    const IT l = rr / rows;
    const IT kw = col % K, ckh = col / K;
    const IT kh = ckh % K, c = ckh / K;
    const IT ow = row % OW, boh = row / OW;
    const IT oh = boh % OH, b = boh / OH;
    const long long h = (long long)(oh * S + kh) - (long long)P, w = (long long)(ow * S + kw) - (long long)P;
    u64 v = 0;
    if (h >= 0 && h < (long long)H && w >= 0 && w < (long long)W)
      v = x[(((i64)(l * B + b) * C + c) * H + h) * (i64)W + w];
    out[t] = v;
  }
}

// Stride 1, K <= 5 (LeNet's 5 x 5): every window gather of an output is
// issued before the sum (predicated loads instead of data-dependent
// continues).
template <int KM>
__global__ void k_col2im_s1(u64* __restrict__ dx, const u64* __restrict__ colsb, uint32_t B, int C, int H, int W,
                            int K, int P, int OH, int OW, uint32_t total, u64 msk) {
  const uint32_t cols = (uint32_t)C * K * K;
  const uint32_t rows = B * (uint32_t)OH * OW;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int w = (int)(t % W);
    const uint32_t t1 = t / W;
    const int h = (int)(t1 % H);
    const uint32_t t2 = t1 / H;
    const int c = (int)(t2 % C);
    const uint32_t bl = t2 / C;
    const uint32_t b = bl % B, l = bl / B;
    const u64* base = colsb + ((i64)l * rows + (i64)b * OH * OW) * cols + (i64)c * K * K;
    u64 v[KM * KM];
#pragma unroll
    for (int kh = 0; kh < KM; ++kh)
#pragma unroll
      for (int kw = 0; kw < KM; ++kw) {
        const int oh = h + P - kh, ow = w + P - kw;
        const bool ok = kh < K && kw < K && oh >= 0 && oh < OH && ow >= 0 && ow < OW;
        v[kh * KM + kw] = ok ? __ldg(base + ((i64)oh * OW + ow) * cols + kh * K + kw) : 0ull;
      }
    u64 acc = 0;
#pragma unroll
    for (int q = 0; q < KM * KM; ++q) acc += v[q];
    dx[t] = acc & msk;
  }
}

template <typename IT, bool S1>
__global__ void k_col2im(u64* __restrict__ dx, const u64* __restrict__ colsb, IT B, IT C, IT H, IT W, IT K,
                         IT S, IT P, IT OH, IT OW, IT total, u64 msk) {
  const IT cols = C * K * K;
  const IT rows = B * OH * OW;
  for (IT t = (IT)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (IT)gridDim.x * blockDim.x) {
    const IT w = t % W;
    const IT t1 = t / W;
    const IT h = t1 % H;
    const IT t2 = t1 / H;
    const IT c = t2 % C;
    const IT bl = t2 / C;
    const IT b = bl % B, l = bl / B;
    u64 acc = 0;
    for (IT kh = 0; kh < K; ++kh) {
      const long long hh = (long long)(h + P) - (long long)kh;
      if (hh < 0 || (!S1 && hh % S)) continue;
      const IT oh = S1 ? (IT)hh : (IT)(hh / S);
      if (oh >= OH) continue;
      for (IT kw = 0; kw < K; ++kw) {
        const long long ww = (long long)(w + P) - (long long)kw;
        if (ww < 0 || (!S1 && ww % S)) continue;
        const IT ow = S1 ? (IT)ww : (IT)(ww / S);
        if (ow >= OW) continue;
        const i64 row = ((i64)b * OH + oh) * OW + ow;
        acc += colsb[((i64)l * rows + row) * cols + ((i64)c * K + kh) * K + kw];
      }
    }
    dx[t] = acc & msk;
  }
}

// Row-per-warp im2col: the (c, kh, kw) -> input-offset table of a column is
// built once per block in shared memory, each warp decodes its output row
// (b, oh, ow) once and its lanes copy the row's columns with coalesced
// stores; no per-element integer division.
__global__ void __launch_bounds__(256) k_im2col_tab(u64* __restrict__ out, const u64* __restrict__ x, int L,
                                                    int B, int C, int H, int W, int K, int S, int P, int OH, int OW) {
  extern __shared__ int tab[];  // [cols] input offset, [cols] kh << 16 | kw
  const int cols = C * K * K;
  for (int col = threadIdx.x; col < cols; col += blockDim.x) {
    const int c = col / (K * K), r = col - c * K * K, kh = r / K, kw = r - kh * K;
    tab[col] = (c * H + kh) * W + kw;
    tab[cols + col] = (kh << 16) | kw;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const i64 rows = (i64)B * OH * OW;
  const i64 nrow = (i64)L * rows;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 lr = warp; lr < nrow; lr += nwarps) {
    const i64 l = lr / rows, row = lr - l * rows;
    const int ow = (int)(row % OW);
    const i64 t = row / OW;
    const int oh = (int)(t % OH);
    const i64 b = t / OH;
    const int h0 = oh * S - P, w0 = ow * S - P;
    const bool inside = h0 >= 0 && w0 >= 0 && h0 + K <= H && w0 + K <= W;
    const u64* xb = x + (l * B + b) * (i64)C * H * W;
    const i64 base = (i64)h0 * W + w0;
    u64* o = out + lr * cols;
    // four columns per lane in flight (the gathers hit L1/L2; one at a time
    // the loop is latency bound)
    for (int c0 = lane; c0 < cols; c0 += 128) {
      u64 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int col = c0 + 32 * q;
        v[q] = 0;
        if (col < cols) {
          if (inside) {
            v[q] = __ldg(xb + base + tab[col]);
          } else {
            const int kk = tab[cols + col], h = h0 + (kk >> 16), w = w0 + (kk & 0xFFFF);
            if (h >= 0 && h < H && w >= 0 && w < W) v[q] = __ldg(xb + base + tab[col]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c0 + 32 * q < cols) o[c0 + 32 * q] = v[q];
    }
  }
}

// Narrow rows (C*K*K < 64, e.g. LeNet conv1's 25 columns): a block owns 256
// consecutive output rows = one contiguous run of 256*cols output words and
// stores it element-per-thread (coalesced); the rows' image offsets and the
// columns' (kh, kw) offsets are decoded once into shared memory, so the
// element loop costs one 32-bit division by cols.
__global__ void __launch_bounds__(256) k_im2col_narrow(u64* __restrict__ out, const u64* __restrict__ x, int L,
                                                       int B, int C, int H, int W, int K, int S, int P, int OH,
                                                       int OW) {
  extern __shared__ i64 nsm[];  // rbase[256] | rhw[256] (int) | tab[cols] | tabk[cols] (int)
  i64* rbase = nsm;
  int* rhw = reinterpret_cast<int*>(nsm + 256);
  int* tab = rhw + 256;
  const int cols = C * K * K;
  int* tabk = tab + cols;
  for (int col = threadIdx.x; col < cols; col += blockDim.x) {
    const int c = col / (K * K), r = col - c * K * K, kh = r / K, kw = r - kh * K;
    tab[col] = (c * H + kh) * W + kw;
    tabk[col] = (kh << 16) | kw;
  }
  const i64 rows = (i64)B * OH * OW, nrow = (i64)L * rows;
  for (i64 r0 = (i64)blockIdx.x * 256; r0 < nrow; r0 += (i64)gridDim.x * 256) {
    __syncthreads();  // previous rows' tables consumed
    const i64 lr = r0 + threadIdx.x;
    if (lr < nrow) {
      const i64 l = lr / rows, row = lr - l * rows;
      const int ow = (int)(row % OW);
      const i64 t = row / OW;
      const int oh = (int)(t % OH);
      const i64 b = t / OH;
      const int h0 = oh * S - P, w0 = ow * S - P;
      rbase[threadIdx.x] = (l * B + b) * (i64)C * H * W + (i64)h0 * W + w0;
      rhw[threadIdx.x] = (int)(((unsigned)(h0 + 0x8000) << 16) | (unsigned)(w0 + 0x8000));
    }
    __syncthreads();
    const int nel = (int)min((i64)256, nrow - r0) * cols;
    u64* o = out + r0 * cols;
    for (int i0 = threadIdx.x; i0 < nel; i0 += 4 * blockDim.x) {
      u64 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = i0 + q * blockDim.x;
        v[q] = 0;
        if (idx < nel) {
          const int rl = idx / cols, col = idx - rl * cols;
          const unsigned hw = (unsigned)rhw[rl];
          const int kk = tabk[col];
          const int h = (int)(hw >> 16) - 0x8000 + (kk >> 16), w = (int)(hw & 0xFFFF) - 0x8000 + (kk & 0xFFFF);
          if (h >= 0 && h < H && w >= 0 && w < W) v[q] = __ldg(x + rbase[rl] + tab[col]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i0 + q * blockDim.x < nel) o[i0 + q * blockDim.x] = v[q];
    }
  }
}

extern "C" int mpx_im2col(uint64_t* out, const uint64_t* x, int L, int64_t B, int C, int H, int W, int K,
                          int stride, int pad, void* stream) {
  CHECK_ARG(out && x && L >= 1 && B >= 1 && C >= 1 && H >= 1 && W >= 1 && K >= 1 && stride >= 1 && pad >= 0);
  const int OH = (H + 2 * pad - K) / stride + 1, OW = (W + 2 * pad - K) / stride + 1;
  CHECK_ARG(OH >= 1 && OW >= 1);
  const i64 total = (i64)L * B * OH * OW * C * K * K;
  if (total == 0) return MPX_OK;
  const i64 cols = (i64)C * K * K;
  // narrow rows (< 64 columns) leave most lanes idle: element-per-thread path
  if (cols >= 64 && cols <= 8192 && (i64)C * H * W < (1ll << 31)) {
    const i64 nrow = (i64)L * B * OH * OW;
    const i64 blocks = min((nrow + 7) / 8, (i64)dev_sms() * 16);
    k_im2col_tab<<<(unsigned)blocks, 256, (size_t)cols * 8, (cudaStream_t)stream>>>(out, x, L, (int)B, C, H, W, K,
                                                                                   stride, pad, OH, OW);
    return launch_status();
  }
  if (cols < 64 && H < 0x4000 && W < 0x4000 && pad < 0x4000) {
    const i64 nrow = (i64)L * B * OH * OW;
    const i64 blocks = min((nrow + 255) / 256, (i64)dev_sms() * 8);
    k_im2col_narrow<<<(unsigned)blocks, 256, 256 * 12 + (size_t)cols * 8, (cudaStream_t)stream>>>(
        out, x, L, (int)B, C, H, W, K, stride, pad, OH, OW);
    return launch_status();
  }
  if (total < (1ll << 31))
    k_im2col<uint32_t><<<grid_for(total), MPX_THREADS, 0, (cudaStream_t)stream>>>(
        out, x, (uint32_t)B, C, H, W, K, stride, pad, OH, OW, (uint32_t)total);
  else
    k_im2col<uint64_t><<<grid_for(total), MPX_THREADS, 0, (cudaStream_t)stream>>>(
        out, x, (uint64_t)B, C, H, W, K, stride, pad, OH, OW, (uint64_t)total);
  return launch_status();
}

extern "C" int mpx_col2im(uint64_t* dx, const uint64_t* cols, int L, int64_t B, int C, int H, int W, int K,
                          int stride, int pad, int width, void* stream) {
  CHECK_ARG(dx && cols && L >= 1 && B >= 1 && C >= 1 && H >= 1 && W >= 1 && K >= 1 && stride >= 1 && pad >= 0 &&
            width >= 1 && width <= 64);
  const int OH = (H + 2 * pad - K) / stride + 1, OW = (W + 2 * pad - K) / stride + 1;
  CHECK_ARG(OH >= 1 && OW >= 1);
  const i64 total = (i64)L * B * C * H * W;
  if (total == 0) return MPX_OK;
  if (stride == 1 && K <= 5 && total < (1ll << 31) && (i64)L * B * OH * OW * C * K * K < (1ll << 31)) {
    k_col2im_s1<5><<<grid_for(total), MPX_THREADS, 0, (cudaStream_t)stream>>>(
        dx, cols, (uint32_t)B, C, H, W, K, pad, OH, OW, (uint32_t)total, ring_mask(width));
    return launch_status();
  }
  if (total < (1ll << 31) && (i64)L * B * OH * OW * C * K * K < (1ll << 32))
    if (stride == 1)
      k_col2im<uint32_t, true><<<grid_for(total), MPX_THREADS, 0, (cudaStream_t)stream>>>(
          dx, cols, (uint32_t)B, C, H, W, K, stride, pad, OH, OW, (uint32_t)total, ring_mask(width));
    else
      k_col2im<uint32_t, false><<<grid_for(total), MPX_THREADS, 0, (cudaStream_t)stream>>>(
          dx, cols, (uint32_t)B, C, H, W, K, stride, pad, OH, OW, (uint32_t)total, ring_mask(width));
  else
    k_col2im<uint64_t, false><<<grid_for(total), MPX_THREADS, 0, (cudaStream_t)stream>>>(
        dx, cols, (uint64_t)B, C, H, W, K, stride, pad, OH, OW, (uint64_t)total, ring_mask(width));
  return launch_status();
}
