// Beaver matrix-product reconstruction in one launch (basic.py:72-75):
//
//   Z_l = C_l + D @ (B_l + [l == p0] E) + A_l @ E        (mod 2^w)
//
// for every local party l, with D = open(X - A), E = open(Y - B). SIMT u64
// tiles for the shapes the tcgen05 limb kernel serves badly: thin outputs
// (N or M far below the 128 x 64 UMMA tile, e.g. a conv layer's 20 output
// channels) and short or very long reductions. Both products share one pass
// over K, the party-0 D @ E term folds into its B operand while the tile is
// staged, and C is read in the epilogue (no separate copy). Tiny outputs
// split K across CTAs and combine with wrapping 64-bit atomics on a copy of C.
#include "common.cuh"

#define BG_BK 16

template <int BM, int BN>
__global__ void __launch_bounds__((BM / 4) * (BN / 4))
    k_beaver_gemm(u64* __restrict__ Z, i64 sZ, const u64* __restrict__ C, i64 sC, const u64* __restrict__ D,
                  const u64* __restrict__ E, const u64* __restrict__ A, i64 sA, const u64* __restrict__ B,
                  i64 sB, int M, int K, int N, int p0, u64 msk, int ksplit, int kchunk) {
  constexpr int TX = BN / 4, TY = BM / 4, NT = TX * TY;
  __shared__ u64 Ds[BG_BK][BM + 1];
  __shared__ u64 As[BG_BK][BM + 1];
  __shared__ u64 Bs[BG_BK][BN];
  __shared__ u64 Es[BG_BK][BN];
  const int l = blockIdx.z / ksplit;
  const int ks = blockIdx.z % ksplit;
  const int kbeg = ks * kchunk, kend = min(K, kbeg + kchunk);
  const u64* Al = A + (i64)l * sA;
  const u64* Bl = B + (i64)l * sB;
  const bool addE = (l == p0);
  const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BN;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  u64 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;

  for (int k0 = kbeg; k0 < kend; k0 += BG_BK) {
#pragma unroll
    for (int q = 0; q < (BM * BG_BK) / NT; ++q) {
      const int idx = threadIdx.x + q * NT;
      const int r = idx / BG_BK, kk = idx % BG_BK;
      const int gr = row0 + r, gk = k0 + kk;
      const bool ok = gr < M && gk < kend;
      const i64 o = (i64)gr * K + gk;
      Ds[kk][r] = ok ? D[o] : 0ull;
      As[kk][r] = ok ? Al[o] : 0ull;
    }
#pragma unroll
    for (int q = 0; q < (BN * BG_BK) / NT; ++q) {
      const int idx = threadIdx.x + q * NT;
      const int kk = idx / BN, c = idx % BN;
      const int gk = k0 + kk, gc = col0 + c;
      const bool ok = gk < kend && gc < N;
      const i64 o = (i64)gk * N + gc;
      const u64 e = ok ? E[o] : 0ull;
      Es[kk][c] = e;
      Bs[kk][c] = ok ? (Bl[o] + (addE ? e : 0ull)) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BG_BK; ++kk) {
      u64 d[4], a[4], b[4], e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        d[i] = Ds[kk][ty + TY * i];
        a[i] = As[kk][ty + TY * i];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        b[j] = Bs[kk][tx + TX * j];
        e[j] = Es[kk][tx + TX * j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += d[i] * b[j] + a[i] * e[j];
    }
    __syncthreads();
  }
  u64* Zl = Z + (i64)l * sZ;
  const u64* Cl = C + (i64)l * sC;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = row0 + ty + TY * i;
    if (gr >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = col0 + tx + TX * j;
      if (gc >= N) continue;
      const i64 o = (i64)gr * N + gc;
      if (ksplit > 1)
        atomicAdd(reinterpret_cast<unsigned long long*>(Zl + o), (unsigned long long)acc[i][j]);
      else
        Zl[o] = (Cl[o] + acc[i][j]) & msk;
    }
  }
}

namespace {
struct Cfg {
  int bm, bn;
};
const Cfg kCfgs[] = {{64, 64}, {128, 32}, {128, 16}, {32, 32}};

template <int BM, int BN>
void launch(dim3 grid, cudaStream_t s, uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* D,
            const uint64_t* E, const uint64_t* A, int64_t sA, const uint64_t* B, int64_t sB, int M, int K, int N,
            int p0, u64 msk, int ksplit, int kchunk) {
  k_beaver_gemm<BM, BN><<<grid, (BM / 4) * (BN / 4), 0, s>>>(Z, sZ, C, sC, D, E, A, sA, B, sB, M, K, N, p0, msk,
                                                              ksplit, kchunk);
}
}  // namespace

extern "C" int mpx_beaver_gemm(uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* D,
                               const uint64_t* E, const uint64_t* A, int64_t sA, const uint64_t* B, int64_t sB,
                               int L, int64_t M, int64_t K, int64_t N, int p0, int width, void* stream) {
  CHECK_ARG(Z && C && D && E && A && B && L >= 1 && M >= 1 && K >= 1 && N >= 1 && width >= 1 && width <= 64);
  CHECK_ARG(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31) && M * K < (1ll << 40));
  CHECK_ARG(p0 < L);
  // tile shape: least padded output area, ties to the larger tile
  int best = 0;
  i64 best_cost = -1;
  for (int c = 0; c < 4; ++c) {
    const i64 bm = kCfgs[c].bm, bn = kCfgs[c].bn;
    const i64 cost = ((M + bm - 1) / bm) * bm * ((N + bn - 1) / bn) * bn;
    if (best_cost < 0 || cost < best_cost) {
      best = c;
      best_cost = cost;
    }
  }
  const int bm = kCfgs[best].bm, bn = kCfgs[best].bn;
  const i64 tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn) * L;
  int ksplit = 1;
  if (width == 64 && tiles < 2 * 148 && K >= 4 * BG_BK) {
    ksplit = (int)min((i64)((2 * 148 + tiles - 1) / tiles), (K + 4 * BG_BK - 1) / (4 * BG_BK));
    if (ksplit < 1) ksplit = 1;
  }
  const i64 kchunk = ((K + ksplit - 1) / ksplit + BG_BK - 1) / BG_BK * BG_BK;
  ksplit = (int)((K + kchunk - 1) / kchunk);
  CHECK_ARG((i64)L * ksplit <= 65535 && (M + bm - 1) / bm <= 65535);
  cudaStream_t s = (cudaStream_t)stream;
  if (ksplit > 1) {
    // every party's partial products land on a copy of its C
    if (cudaMemcpy2DAsync(Z, (size_t)sZ * 8, C, (size_t)sC * 8, (size_t)(M * N * 8), (size_t)L,
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return MPX_ERR_CUDA;
  }
  dim3 grid((unsigned)((N + bn - 1) / bn), (unsigned)((M + bm - 1) / bm), (unsigned)(L * ksplit));
  const u64 msk = ring_mask(width);
  switch (best) {
    case 0: launch<64, 64>(grid, s, Z, sZ, C, sC, D, E, A, sA, B, sB, (int)M, (int)K, (int)N, p0, msk, ksplit, (int)kchunk); break;
    case 1: launch<128, 32>(grid, s, Z, sZ, C, sC, D, E, A, sA, B, sB, (int)M, (int)K, (int)N, p0, msk, ksplit, (int)kchunk); break;
    case 2: launch<128, 16>(grid, s, Z, sZ, C, sC, D, E, A, sA, B, sB, (int)M, (int)K, (int)N, p0, msk, ksplit, (int)kchunk); break;
    default: launch<32, 32>(grid, s, Z, sZ, C, sC, D, E, A, sA, B, sB, (int)M, (int)K, (int)N, p0, msk, ksplit, (int)kchunk); break;
  }
  return launch_status();
}
