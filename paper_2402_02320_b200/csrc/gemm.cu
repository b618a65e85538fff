// Z_2^64 matrix products (ring.py:60-62; basic.py:72-75; preprocessing.py:150;
// nn.py:193).
//
// mpx_gemm dispatches between:
//  * gemm_u64_simt: exact 64-bit SIMT tiles (64x64 per CTA, 4x4 per thread),
//    used for small / skinny products and as the general fallback shape;
//  * the tcgen05 int8-limb kernel (gemm_tc.cu) for large products, where
//    A and B are split into 8 byte limbs and the 36 limb products with
//    i + j <= 7 are accumulated per diagonal in TMEM.
#include "common.cuh"

#define GT_BM 64
#define GT_BN 64
#define GT_BK 16

__global__ void __launch_bounds__(256) gemm_u64_simt(u64* __restrict__ C, const u64* __restrict__ A,
                                                     const u64* __restrict__ B, i64 M, i64 K, i64 N,
                                                     i64 sA, i64 sB, i64 sC, int accumulate, u64 msk,
                                                     int ksplit, i64 kchunk) {
  __shared__ u64 As[GT_BK][GT_BM + 1];
  __shared__ u64 Bs[GT_BK][GT_BN];
  const i64 bz = blockIdx.z / ksplit;
  const int ks = blockIdx.z % ksplit;
  const i64 kbeg = ks * kchunk, kend = min(K, kbeg + kchunk);
  A += bz * sA;
  B += bz * sB;
  C += bz * sC;
  const i64 row0 = (i64)blockIdx.y * GT_BM;
  const i64 col0 = (i64)blockIdx.x * GT_BN;
  const int tx = threadIdx.x & 15;  // column group
  const int ty = threadIdx.x >> 4;  // row group
  u64 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;

  for (i64 k0 = kbeg; k0 < kend; k0 += GT_BK) {
    // A tile: 64 rows x 16 k = 1024 values, 4 per thread (k fastest for coalescing)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + q * 256;
      const int r = idx / GT_BK, kk = idx % GT_BK;
      const i64 gr = row0 + r, gk = k0 + kk;
      As[kk][r] = (gr < M && gk < kend) ? A[gr * K + gk] : 0ull;
    }
    // B tile: 16 k x 64 cols
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + q * 256;
      const int kk = idx / GT_BN, c = idx % GT_BN;
      const i64 gk = k0 + kk, gc = col0 + c;
      Bs[kk][c] = (gk < kend && gc < N) ? B[gk * N + gc] : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GT_BK; ++kk) {
      u64 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const i64 gr = row0 + ty + 16 * i;
    if (gr >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const i64 gc = col0 + tx + 16 * j;
      if (gc >= N) continue;
      if (ksplit > 1) {
        atomicAdd(reinterpret_cast<unsigned long long*>(C + gr * N + gc), (unsigned long long)acc[i][j]);
      } else {
        u64 v = acc[i][j];
        if (accumulate) v += C[gr * N + gc];
        C[gr * N + gc] = v & msk;
      }
    }
  }
}

// Implemented in gemm_tc.cu; returns MPX_ERR_UNSUPPORTED when the shape is
// not served by the tensor-core path.
int mpx_gemm_tc(uint64_t* C, const uint64_t* A, const uint64_t* B, int64_t batch, int64_t M, int64_t K,
                int64_t N, int64_t sA, int64_t sB, int64_t sC, int accumulate, int width, cudaStream_t s);

extern "C" int mpx_gemm_simt(uint64_t* C, const uint64_t* A, const uint64_t* B, int64_t batch, int64_t M,
                             int64_t K, int64_t N, int64_t sA, int64_t sB, int64_t sC, int accumulate,
                             int width, void* stream) {
  CHECK_ARG(C && A && B && batch >= 1 && M >= 0 && K >= 0 && N >= 0 && width >= 1 && width <= 64);
  CHECK_ARG(batch <= 65535);
  if (M == 0 || N == 0) return MPX_OK;
  const i64 tiles = ((N + GT_BN - 1) / GT_BN) * ((M + GT_BM - 1) / GT_BM) * batch;
  // split K across CTAs when the output grid cannot fill the SMs (width 64:
  // partial sums combine with wrapping 64-bit atomics)
  int ksplit = 1;
  if (width == 64 && tiles < 2 * dev_sms() && K >= 4 * GT_BK) {
    ksplit = (int)min((i64)(2 * dev_sms() / tiles), (K + 2 * GT_BK - 1) / (2 * GT_BK));
    if (ksplit < 1) ksplit = 1;
  }
  const i64 kchunk = ((K + ksplit - 1) / ksplit + GT_BK - 1) / GT_BK * GT_BK;
  ksplit = (int)((K + kchunk - 1) / kchunk);
  CHECK_ARG(batch * ksplit <= 65535);
  cudaStream_t st = (cudaStream_t)stream;
  if (ksplit > 1 && !accumulate)
    for (i64 z = 0; z < batch; ++z)
      if (cudaMemsetAsync(C + z * sC, 0, (size_t)(M * N * 8), st) != cudaSuccess) return MPX_ERR_CUDA;
  dim3 grid((unsigned)((N + GT_BN - 1) / GT_BN), (unsigned)((M + GT_BM - 1) / GT_BM), (unsigned)(batch * ksplit));
  CHECK_ARG(grid.y <= 65535);
  gemm_u64_simt<<<grid, 256, 0, st>>>(C, A, B, M, K, N, sA, sB, sC, accumulate, ring_mask(width), ksplit,
                                      ksplit > 1 ? kchunk : K);
  return launch_status();
}

extern "C" int mpx_gemm(uint64_t* C, const uint64_t* A, const uint64_t* B, int64_t batch, int64_t M,
                        int64_t K, int64_t N, int64_t sA, int64_t sB, int64_t sC, int accumulate, int width,
                        void* stream) {
  int rc = mpx_gemm_tc(C, A, B, batch, M, K, N, sA, sB, sC, accumulate, width, (cudaStream_t)stream);
  if (rc != MPX_ERR_UNSUPPORTED) return rc;
  return mpx_gemm_simt(C, A, B, batch, M, K, N, sA, sB, sC, accumulate, width, stream);
}
