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
#include <stdlib.h>

#include "common.cuh"

#define BG_BK 16


// Z[b][l] = C[b][l] (M*N words each) for every product b and party l: the
// split-K partial products then land on a copy of C. One 2D copy when the
// (product, party) slabs sit at uniform pitches; else one per party (rows =
// products) or one per product (rows = parties), whichever is fewer.
static int batch_copy_c(u64* Z, i64 sZ, i64 bZ, const u64* C, i64 sC, i64 bC, i64 MN, int L, i64 batch,
                        cudaStream_t s) {
  const size_t w = (size_t)(MN * 8);
  if (batch == 1 || (bZ == (i64)L * sZ && bC == (i64)L * sC))
    return cudaMemcpy2DAsync(Z, (size_t)sZ * 8, C, (size_t)sC * 8, w, (size_t)(L * batch), cudaMemcpyDeviceToDevice,
                             s) == cudaSuccess ? MPX_OK : MPX_ERR_CUDA;
  if (L < batch && bZ >= MN && bC >= MN) {
    for (int l = 0; l < L; ++l)
      if (cudaMemcpy2DAsync(Z + l * sZ, (size_t)bZ * 8, C + l * sC, (size_t)bC * 8, w, (size_t)batch,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return MPX_ERR_CUDA;
    return MPX_OK;
  }
  for (i64 b = 0; b < batch; ++b)
    if (cudaMemcpy2DAsync(Z + b * bZ, (size_t)sZ * 8, C + b * bC, (size_t)sC * 8, w, (size_t)L,
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return MPX_ERR_CUDA;
  return MPX_OK;
}

// <= 128 registers per thread (a block occupies whole warps)
constexpr int bg_min_blocks(int nt) { return 512 / (nt < 32 ? 32 : nt); }

template <int BM, int BN, int TN, bool FULL, int KB = BG_BK>
__device__ __forceinline__ void bg_tile_math(u64 (&acc)[4][TN], const u64 (*Ds)[BM + 1], const u64 (*As)[BM + 1],
                                             const u64 (*Bs)[BN], const u64 (*Es)[BN], int tx, int ty, int kn,
                                             bool addE) {
  constexpr int TX = BN / TN, TY = BM / 4;
#pragma unroll
  for (int kk = 0; kk < KB; ++kk) {
    if (!FULL && kk >= kn) break;
    u64 d[4], a[4], b[TN], e[TN];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      d[i] = Ds[kk][ty + TY * i];
      a[i] = As[kk][ty + TY * i];
    }
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      e[j] = Es[kk][tx + TX * j];
      b[j] = Bs[kk][tx + TX * j] + (addE ? e[j] : 0ull);  // party 0's B' = B + E (basic.py:72-75)
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] += d[i] * b[j] + a[i] * e[j];
  }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool ok) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(ok ? 8 : 0) : "memory");
}

template <int BM, int BN>
constexpr int bg_stage_words() {
  return 2 * BG_BK * (BM + 1) + 2 * BG_BK * BN;
}

// CTA tile BM x BN, each thread 4 rows x TN columns (strided by TY / TX so
// shared-memory reads are conflict-free broadcasts / consecutive words). The
// operand tiles stream through a two-stage cp.async pipeline (the next k-step
// is in flight while this one multiplies).
template <int BM, int BN, int TN>
__global__ void __launch_bounds__((BM / 4) * (BN / TN), bg_min_blocks((BM / 4) * (BN / TN)))
    k_beaver_gemm(u64* __restrict__ Z, i64 sZ, const u64* __restrict__ C, i64 sC, const u64* __restrict__ D,
                  const u64* __restrict__ E, const u64* __restrict__ A, i64 sA, const u64* __restrict__ B,
                  i64 sB, int M, int K, int N, int p0, u64 msk, int ksplit, int kchunk, int L, i64 bZ, i64 bC,
                  i64 bA, i64 bB) {
  constexpr int TX = BN / TN, TY = BM / 4, NT = TX * TY;
  constexpr int STAGE = bg_stage_words<BM, BN>();
  extern __shared__ u64 bg_sm[];
  typedef u64 RowM[BM + 1];
  typedef u64 RowN[BN];
  auto Ds = [&](int s) { return reinterpret_cast<RowM*>(bg_sm + s * STAGE); };
  auto As = [&](int s) { return reinterpret_cast<RowM*>(bg_sm + s * STAGE + BG_BK * (BM + 1)); };
  auto Bs = [&](int s) { return reinterpret_cast<RowN*>(bg_sm + s * STAGE + 2 * BG_BK * (BM + 1)); };
  auto Es = [&](int s) { return reinterpret_cast<RowN*>(bg_sm + s * STAGE + 2 * BG_BK * (BM + 1) + BG_BK * BN); };
  const int zl = blockIdx.z / ksplit;  // (product, party)
  const int ks = blockIdx.z % ksplit;
  const int bt = zl / L, l = zl - bt * L;
  Z += bt * bZ;
  C += bt * bC;
  A += bt * bA;
  B += bt * bB;
  D += (i64)bt * M * K;
  E += (i64)bt * K * N;
  const int kbeg = ks * kchunk, kend = min(K, kbeg + kchunk);
  const u64* Al = A + (i64)l * sA;
  const u64* Bl = B + (i64)l * sB;
  const bool addE = (l == p0);
  const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BN;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  u64 acc[4][TN];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0;

  auto issue = [&](int s, int k0) {
    RowM* ds = Ds(s);
    RowM* as = As(s);
    RowN* bs = Bs(s);
    RowN* es = Es(s);
    for (int idx = threadIdx.x; idx < BM * BG_BK; idx += NT) {
      const int r = idx / BG_BK, kk = idx % BG_BK;
      const int gr = row0 + r, gk = k0 + kk;
      const bool ok = gr < M && gk < kend;
      const i64 o = ok ? (i64)gr * K + gk : 0;
      cp_async8(&ds[kk][r], D + o, ok);
      cp_async8(&as[kk][r], Al + o, ok);
    }
    for (int idx = threadIdx.x; idx < BN * BG_BK; idx += NT) {
      const int kk = idx / BN, c = idx % BN;
      const int gk = k0 + kk, gc = col0 + c;
      const bool ok = gk < kend && gc < N;
      const i64 o = ok ? (i64)gk * N + gc : 0;
      cp_async8(&es[kk][c], E + o, ok);
      cp_async8(&bs[kk][c], Bl + o, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int nsteps = kend > kbeg ? (kend - kbeg + BG_BK - 1) / BG_BK : 0;
  if (nsteps > 0) issue(0, kbeg);
  for (int step = 0; step < nsteps; ++step) {
    const int k0 = kbeg + step * BG_BK;
    if (step + 1 < nsteps) {
      issue((step + 1) & 1, k0 + BG_BK);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int s = step & 1;
    const int kn = kend - k0;
    if (kn >= BG_BK)
      bg_tile_math<BM, BN, TN, true>(acc, Ds(s), As(s), Bs(s), Es(s), tx, ty, kn, addE);
    else
      bg_tile_math<BM, BN, TN, false>(acc, Ds(s), As(s), Bs(s), Es(s), tx, ty, kn, addE);
    __syncthreads();
  }
  u64* Zl = Z + (i64)l * sZ;
  const u64* Cl = C + (i64)l * sC;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = row0 + ty + TY * i;
    if (gr >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
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
  int bm, bn, tn;
};
// (BM, BN, TN): square-ish tiles for wide outputs, thin ones sized to common
// layer widths (20 / 10 output channels), small-M tiles for weight gradients
const Cfg kCfgs[] = {{64, 64, 4}, {128, 32, 4}, {128, 16, 4}, {32, 32, 4},
                     {128, 20, 5}, {128, 10, 5}, {32, 20, 5}, {32, 10, 5}};
constexpr int kNumCfgs = sizeof(kCfgs) / sizeof(kCfgs[0]);

struct Batch {
  int L;
  i64 bZ, bC, bA, bB;
};

template <int BM, int BN, int TN>
int launch(dim3 grid, cudaStream_t s, uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* D,
           const uint64_t* E, const uint64_t* A, int64_t sA, const uint64_t* B, int64_t sB, int M, int K, int N,
           int p0, u64 msk, int ksplit, int kchunk, const Batch& bt) {
  constexpr int smem = 2 * bg_stage_words<BM, BN>() * 8;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_beaver_gemm<BM, BN, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return MPX_ERR_CUDA;
    attr = true;
  }
  k_beaver_gemm<BM, BN, TN><<<grid, (BM / 4) * (BN / TN), smem, s>>>(Z, sZ, C, sC, D, E, A, sA, B, sB, M, K, N, p0,
                                                                       msk, ksplit, kchunk, bt.L, bt.bZ, bt.bC,
                                                                       bt.bA, bt.bB);
  return MPX_OK;
}
}  // namespace

extern "C" int mpx_beaver_gemm_batched(uint64_t* Z, int64_t sZ, int64_t bZ, const uint64_t* C, int64_t sC,
                                       int64_t bC, const uint64_t* D, const uint64_t* E, const uint64_t* A,
                                       int64_t sA, int64_t bA, const uint64_t* B, int64_t sB, int64_t bB, int L,
                                       int64_t batch, int64_t M, int64_t K, int64_t N, int p0, int width,
                                       void* stream) {
  CHECK_ARG(Z && C && D && E && A && B && L >= 1 && M >= 1 && K >= 1 && N >= 1 && width >= 1 && width <= 64);
  CHECK_ARG(batch >= 1 && batch * L <= 65535);
  const Batch bt{L, bZ, bC, bA, bB};
  CHECK_ARG(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31) && M * K < (1ll << 40));
  CHECK_ARG(p0 < L);
  // tile shape: least padded output area, ties to the larger tile
  int best = 0;
  i64 best_cost = -1, best_area = 0;
  for (int c = 0; c < kNumCfgs; ++c) {
    const i64 bm = kCfgs[c].bm, bn = kCfgs[c].bn;
    const i64 cost = ((M + bm - 1) / bm) * bm * ((N + bn - 1) / bn) * bn;
    if (best_cost < 0 || cost < best_cost || (cost == best_cost && bm * bn > best_area)) {
      best = c;
      best_cost = cost;
      best_area = bm * bn;
    }
  }
  const int bm = kCfgs[best].bm, bn = kCfgs[best].bn;
  const int nt = (bm / 4) * (bn / kCfgs[best].tn);
  const i64 tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn) * L * batch;
  // resident CTAs per SM at <= 128 registers per thread
  i64 per_sm = min((i64)32, (i64)(65536 / (max(nt, 32) * 128)));
  if (const char* cap = getenv("MPX_BG_PER_SM")) per_sm = min(per_sm, (i64)max(1, atoi(cap)));  // sweeps
  const i64 target = (i64)dev_sms() * per_sm;
  int ksplit = 1;
  if (width == 64 && tiles < target && K >= 4 * BG_BK) {
    ksplit = (int)min((target + tiles - 1) / tiles, (K + BG_BK - 1) / BG_BK);
    if (ksplit < 1) ksplit = 1;
  }
  const i64 kchunk = ((K + ksplit - 1) / ksplit + BG_BK - 1) / BG_BK * BG_BK;
  ksplit = (int)((K + kchunk - 1) / kchunk);
  CHECK_ARG((i64)L * batch * ksplit <= 65535 && (M + bm - 1) / bm <= 65535);
  cudaStream_t s = (cudaStream_t)stream;
  if (ksplit > 1) {
    // every party's partial products land on a copy of its C
    if (batch_copy_c(Z, sZ, bZ, C, sC, bC, (i64)M * N, L, batch, s) != MPX_OK) return MPX_ERR_CUDA;
  }
  dim3 grid((unsigned)((N + bn - 1) / bn), (unsigned)((M + bm - 1) / bm), (unsigned)(L * batch * ksplit));
  const u64 msk = ring_mask(width);
#define BG_CASE(I, BM_, BN_, TN_)                                                                             \
  case I:                                                                                                    \
    if (launch<BM_, BN_, TN_>(grid, s, Z, sZ, C, sC, D, E, A, sA, B, sB, (int)M, (int)K, (int)N, p0, msk,     \
                              ksplit, (int)kchunk, bt) != MPX_OK)                                            \
      return MPX_ERR_CUDA;                                                                                   \
    break;
  switch (best) {
    BG_CASE(0, 64, 64, 4)
    BG_CASE(1, 128, 32, 4)
    BG_CASE(2, 128, 16, 4)
    BG_CASE(3, 32, 32, 4)
    BG_CASE(4, 128, 20, 5)
    BG_CASE(5, 128, 10, 5)
    BG_CASE(6, 32, 20, 5)
    default: BG_CASE(7, 32, 10, 5)
  }
#undef BG_CASE
  return launch_status();
}

extern "C" int mpx_beaver_gemm(uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* D,
                               const uint64_t* E, const uint64_t* A, int64_t sA, const uint64_t* B, int64_t sB,
                               int L, int64_t M, int64_t K, int64_t N, int p0, int width, void* stream) {
  return mpx_beaver_gemm_batched(Z, sZ, 0, C, sC, 0, D, E, A, sA, 0, B, sB, 0, L, 1, M, K, N, p0, width, stream);
}

// ---------------------------------------------------------------------------
// All parties local (sim sessions): the Beaver opening folded into the
// product. D = sum_l (X_l - A_l) and E = sum_l (Y_l - B_l) (basic.py:66-70,
// an opening is a sum over the party axis) are formed tile by tile in shared
// memory next to every party's A_l / B_l tile, and the CTA's L party groups
// (NT threads each) reconstruct Z_l = C_l + D @ (B_l + [l==p0] E) + A_l @ E
// from them. One launch replaces mask(D) + mask(E) + reconstruct; D and E
// never reach HBM, and the operands are read once for all parties. X / Y are
// logical M x K / K x N share views at any (party, row, col) strides (the
// transposed im2col / activation views are read in place); material A_l,
// B_l is row-major. Shared-memory fills walk each source along its unit
// stride.
struct SimOperand {
  const u64* p;
  i64 ps, sr, sc, js;  // party, row, col, job strides (elements)
};

#ifndef BS_BK
#define BS_BK 8  // k-depth of one pipeline stage
#endif

// Raw operand tiles of one k-step: every party's X_l, A_l, Y_l, B_l.
template <int L, int BM, int BN>
constexpr int bs_stage_words() {
  return 2 * L * BS_BK * (BM + 1) + 2 * L * BS_BK * BN;
}

template <int L, int BM, int BN, int TN>
__global__ void __launch_bounds__(L*(BM / 4) * (BN / TN))
    k_beaver_gemm_sim(u64* __restrict__ Z, i64 sZ, i64 bZ, const u64* __restrict__ C, i64 sC, i64 bC,
                      const __grid_constant__ SimOperand X, const u64* __restrict__ A, i64 sA, i64 bA,
                      const __grid_constant__ SimOperand Y, const u64* __restrict__ B, i64 sB, i64 bB, int M,
                      int K, int N, int p0, u64 msk, int ksplit, int kchunk) {
  constexpr int TX = BN / TN, TY = BM / 4, NT = TX * TY, NTL = L * NT;
  constexpr int STAGE = bs_stage_words<L, BM, BN>();
  typedef u64 RowM[BM + 1];
  typedef u64 RowN[BN];
  extern __shared__ u64 bs_sm[];
  // stage s: Xs[L][BK] | As[L][BK] (RowM), Ys[L][BK] | Bs[L][BK] (RowN); then D[BK] (RowM), E[BK] (RowN)
  auto Xs = [&](int st) { return reinterpret_cast<RowM*>(bs_sm + st * STAGE); };
  auto As = [&](int st) { return reinterpret_cast<RowM*>(bs_sm + st * STAGE) + L * BS_BK; };
  auto Ys = [&](int st) { return reinterpret_cast<RowN*>(bs_sm + st * STAGE + 2 * L * BS_BK * (BM + 1)); };
  auto Bs = [&](int st) { return Ys(st) + L * BS_BK; };
  RowM* Ds = reinterpret_cast<RowM*>(bs_sm + 2 * STAGE);
  RowN* Es = reinterpret_cast<RowN*>(bs_sm + 2 * STAGE + BS_BK * (BM + 1));
  const int bt = blockIdx.z / ksplit, ks = blockIdx.z % ksplit;
  Z += bt * bZ;
  C += bt * bC;
  A += bt * bA;
  B += bt * bB;
  const u64* Xp = X.p + bt * X.js;
  const u64* Yp = Y.p + bt * Y.js;
  const int kbeg = ks * kchunk, kend = min(K, kbeg + kchunk);
  const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BN;
  const int tid = threadIdx.x, l = tid / NT, t = tid % NT;
  const int tx = t % TX, ty = t / TX;
  const bool xrow = X.sc == 1, yrow = Y.sc == 1;  // k (resp. n) is X's (Y's) unit stride
  u64 acc[4][TN];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0;

  // cp.async of one k-step's raw tiles (zero-filled outside the matrices);
  // each source is walked along its unit stride
  auto issue = [&](int st, int k0) {
    RowM* xs = Xs(st);
    RowM* as = As(st);
    RowN* ys = Ys(st);
    RowN* bs = Bs(st);
    for (int idx = tid; idx < BM * BS_BK; idx += NTL) {
      const int r = idx / BS_BK, kk = idx % BS_BK, gr = row0 + r, gk = k0 + kk;
      const bool ok = gr < M && gk < kend;
      const u64* src = A + (ok ? (i64)gr * K + gk : 0);
#pragma unroll
      for (int q = 0; q < L; ++q) cp_async8(&as[q * BS_BK + kk][r], src + (ok ? q * sA : 0), ok);
    }
    for (int idx = tid; idx < BM * BS_BK; idx += NTL) {
      const int r = xrow ? idx / BS_BK : idx % BM, kk = xrow ? idx % BS_BK : idx / BM;
      const int gr = row0 + r, gk = k0 + kk;
      const bool ok = gr < M && gk < kend;
      const u64* src = Xp + (ok ? (i64)gr * X.sr + (i64)gk * X.sc : 0);
#pragma unroll
      for (int q = 0; q < L; ++q) cp_async8(&xs[q * BS_BK + kk][r], src + (ok ? q * X.ps : 0), ok);
    }
    for (int idx = tid; idx < BN * BS_BK; idx += NTL) {
      const int kk = idx / BN, c = idx % BN, gk = k0 + kk, gc = col0 + c;
      const bool ok = gk < kend && gc < N;
      const u64* src = B + (ok ? (i64)gk * N + gc : 0);
#pragma unroll
      for (int q = 0; q < L; ++q) cp_async8(&bs[q * BS_BK + kk][c], src + (ok ? q * sB : 0), ok);
    }
    for (int idx = tid; idx < BN * BS_BK; idx += NTL) {
      const int c = yrow ? idx % BN : idx / BS_BK, kk = yrow ? idx / BN : idx % BS_BK;
      const int gk = k0 + kk, gc = col0 + c;
      const bool ok = gk < kend && gc < N;
      const u64* src = Yp + (ok ? (i64)gk * Y.sr + (i64)gc * Y.sc : 0);
#pragma unroll
      for (int q = 0; q < L; ++q) cp_async8(&ys[q * BS_BK + kk][c], src + (ok ? q * Y.ps : 0), ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int nsteps = kend > kbeg ? (kend - kbeg + BS_BK - 1) / BS_BK : 0;
  if (nsteps > 0) issue(0, kbeg);
  for (int step = 0; step < nsteps; ++step) {
    const int k0 = kbeg + step * BS_BK, st = step & 1;
    if (step + 1 < nsteps) {
      issue(st ^ 1, k0 + BS_BK);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    {  // the opening: D = sum_l X_l - A_l, E = sum_l Y_l - B_l of this k-step
      const RowM* xs = Xs(st);
      const RowM* as = As(st);
      const RowN* ys = Ys(st);
      const RowN* bs = Bs(st);
      for (int idx = tid; idx < BM * BS_BK; idx += NTL) {
        const int kk = idx / BM, r = idx % BM;
        u64 d = 0;
#pragma unroll
        for (int q = 0; q < L; ++q) d += xs[q * BS_BK + kk][r] - as[q * BS_BK + kk][r];
        Ds[kk][r] = d;
      }
      for (int idx = tid; idx < BN * BS_BK; idx += NTL) {
        const int kk = idx / BN, c = idx % BN;
        u64 e = 0;
#pragma unroll
        for (int q = 0; q < L; ++q) e += ys[q * BS_BK + kk][c] - bs[q * BS_BK + kk][c];
        Es[kk][c] = e;
      }
    }
    __syncthreads();
    const int kn = kend - k0;
    if (kn >= BS_BK)
      bg_tile_math<BM, BN, TN, true, BS_BK>(acc, Ds, As(st) + l * BS_BK, Bs(st) + l * BS_BK, Es, tx, ty, kn,
                                            l == p0);
    else
      bg_tile_math<BM, BN, TN, false, BS_BK>(acc, Ds, As(st) + l * BS_BK, Bs(st) + l * BS_BK, Es, tx, ty, kn,
                                             l == p0);
    __syncthreads();
  }
  u64* Zl = Z + (i64)l * sZ;
  const u64* Cl = C + (i64)l * sC;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = row0 + ty + TY * i;
    if (gr >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
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
template <int L, int BM, int BN>
constexpr int bs_smem_bytes() {
  return 8 * (2 * bs_stage_words<L, BM, BN>() + BS_BK * (BM + 1 + BN));
}

template <int L, int BM, int BN, int TN>
int launch_sim(i64 tiles_n, i64 tiles_m, i64 batch, i64 K, cudaStream_t s, uint64_t* Z, int64_t sZ, int64_t bZ,
               const uint64_t* C, int64_t sC, int64_t bC, const SimOperand& X, const uint64_t* A, int64_t sA,
               int64_t bA, const SimOperand& Y, const uint64_t* B, int64_t sB, int64_t bB, int M, int N, int p0,
               int width) {
  constexpr int smem = bs_smem_bytes<L, BM, BN>();
  constexpr int nthr = L * (BM / 4) * (BN / TN);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_beaver_gemm_sim<L, BM, BN, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess)
      return MPX_ERR_CUDA;
    attr = true;
  }
  // resident CTAs per SM of this instantiation: split K to fill exactly one wave
  static int occ = 0;
  if (!occ && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_beaver_gemm_sim<L, BM, BN, TN>, nthr, smem) !=
                   cudaSuccess ||
               occ < 1))
    occ = 1;
  i64 per_sm = occ;
  if (const char* ov = getenv("MPX_BS_PER_SM")) per_sm = max(1, atoi(ov));  // sweeps
  const i64 tiles = tiles_n * tiles_m * batch, target = (i64)dev_sms() * per_sm;
  int ksplit = 1;
  if (width == 64 && tiles < target && K >= 4 * BS_BK)
    ksplit = (int)max((i64)1, min((target + tiles - 1) / tiles, (K + 2 * BS_BK - 1) / (2 * BS_BK)));
  const i64 kchunk = ((K + ksplit - 1) / ksplit + BS_BK - 1) / BS_BK * BS_BK;
  ksplit = (int)((K + kchunk - 1) / kchunk);
  if (batch * ksplit > 65535 || tiles_m > 65535) return MPX_ERR_ARG;
  if (ksplit > 1) {
    if (batch_copy_c(Z, sZ, bZ, C, sC, bC, (i64)M * N, L, batch, s) != MPX_OK) return MPX_ERR_CUDA;
  }
  dim3 grid((unsigned)tiles_n, (unsigned)tiles_m, (unsigned)(batch * ksplit));
  k_beaver_gemm_sim<L, BM, BN, TN><<<grid, nthr, smem, s>>>(Z, sZ, bZ, C, sC, bC, X, A, sA, bA, Y, B, sB, bB, M,
                                                            (int)K, N, p0, ring_mask(width), ksplit, (int)kchunk);
  return launch_status();
}

// tiles with at most 128 threads per party group
const Cfg kSimCfgs[] = {{32, 32, 4}, {64, 32, 4}, {128, 16, 4}, {128, 20, 5}, {128, 10, 5}, {32, 20, 5}, {32, 10, 5}};
constexpr int kNumSimCfgs = sizeof(kSimCfgs) / sizeof(kSimCfgs[0]);

template <int L>
int dispatch_sim(int best, i64 K, i64 batch, cudaStream_t s, uint64_t* Z, int64_t sZ, int64_t bZ, const uint64_t* C,
                 int64_t sC, int64_t bC, const SimOperand& X, const uint64_t* A, int64_t sA, int64_t bA,
                 const SimOperand& Y, const uint64_t* B, int64_t sB, int64_t bB, int M, int N, int p0, int width) {
#define BS_CASE(I, BM_, BN_, TN_)                                                                              \
  case I:                                                                                                     \
    return launch_sim<L, BM_, BN_, TN_>((N + BN_ - 1) / BN_, (M + BM_ - 1) / BM_, batch, K, s, Z, sZ, bZ, C, sC, \
                                        bC, X, A, sA, bA, Y, B, sB, bB, M, N, p0, width);
  switch (best) {
    BS_CASE(0, 32, 32, 4)
    BS_CASE(1, 64, 32, 4)
    BS_CASE(2, 128, 16, 4)
    BS_CASE(3, 128, 20, 5)
    BS_CASE(4, 128, 10, 5)
    BS_CASE(5, 32, 20, 5)
    default:
      BS_CASE(6, 32, 10, 5)
  }
#undef BS_CASE
}
}  // namespace

// --------------------------------------------------------------------------
// Tall thin sim-mode products (all parties local): huge M, K <= 32, N <= 32
// (a first conv layer's forward product, 73728 x 25 x 20 at LeNet batch
// 128), which the tiled kernel above serves with too few threads per SM.
// Each CTA holds E and every party's B' = B_l + [l==p0] E for the whole
// (tiny) K x N in shared memory, then streams 32-row groups: the rows'
// X_l / A_l words are read once (contiguous), D = sum_l X_l - A_l is formed
// in shared memory, and warp l / lane r computes party l's output row r
// against B'_l and E. (A long-K / tiny-output variant for the weight
// gradient measured slower than the tiled split-K kernel: 158 vs 127 us.)

#define TALL_R 32

template <int L, int NT>
__global__ void __launch_bounds__(32 * L) k_beaver_tall(u64* __restrict__ Z, i64 sZ, i64 bZ, const u64* __restrict__ C,
                                                        i64 sC, i64 bC, const __grid_constant__ SimOperand X,
                                                        const u64* __restrict__ A, i64 sA, i64 bA,
                                                        const __grid_constant__ SimOperand Y,
                                                        const u64* __restrict__ B, i64 sB, i64 bB, int M, int K,
                                                        int N, int p0, u64 msk) {
  extern __shared__ __align__(16) u64 tl_sm[];
  const int KP = K | 1;                       // odd row pitch: conflict-free per-row reads
  u64* Bp = tl_sm;                            // [L][K][NT]
  u64* Es = Bp + L * K * NT;                  // [K][NT]
  u64* Ds = Es + K * NT;                      // [TALL_R][KP]
  u64* As = Ds + TALL_R * KP;                 // [L][TALL_R][KP]
  const int bt = blockIdx.y;
  Z += bt * bZ;
  C += bt * bC;
  A += bt * bA;
  B += bt * bB;
  const u64* Xp = X.p + bt * X.js;
  const u64* Yp = Y.p + bt * Y.js;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int idx = tid; idx < K * NT; idx += nt) {
    const int k = idx / NT, j = idx % NT;
    u64 e = 0;
    u64 b[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
      b[l] = j < N ? B[l * sB + (i64)k * N + j] : 0ull;
      e += (j < N ? Yp[l * Y.ps + (i64)k * Y.sr + (i64)j * Y.sc] : 0ull) - b[l];
    }
    Es[k * NT + j] = e;
#pragma unroll
    for (int l = 0; l < L; ++l) Bp[(l * K + k) * NT + j] = b[l] + (l == p0 ? e : 0ull);
  }
  const int l = tid >> 5, r = tid & 31;
  for (i64 r0 = (i64)blockIdx.x * TALL_R; r0 < M; r0 += (i64)gridDim.x * TALL_R) {
    __syncthreads();  // E / B' ready; previous group's rows consumed
    for (int idx = tid; idx < TALL_R * K; idx += nt) {
      const int rr = idx / K, k = idx % K;
      const i64 gr = r0 + rr;
      u64 d = 0;
#pragma unroll
      for (int q = 0; q < L; ++q) {
        const u64 x = gr < M ? Xp[q * X.ps + gr * X.sr + (i64)k * X.sc] : 0ull;
        const u64 a = gr < M ? A[q * sA + gr * K + k] : 0ull;
        As[(q * TALL_R + rr) * KP + k] = a;
        d += x - a;
      }
      Ds[rr * KP + k] = d;
    }
    __syncthreads();
    u64 acc[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j] = 0;
    const u64* bl = Bp + l * K * NT;
    for (int k = 0; k < K; ++k) {
      const u64 d = Ds[r * KP + k], a = As[(l * TALL_R + r) * KP + k];
      const ulonglong2* b2 = reinterpret_cast<const ulonglong2*>(bl + k * NT);
      const ulonglong2* e2 = reinterpret_cast<const ulonglong2*>(Es + k * NT);
#pragma unroll
      for (int j = 0; j < NT / 2; ++j) {
        const ulonglong2 bb = b2[j], ee = e2[j];
        acc[2 * j] += d * bb.x + a * ee.x;
        acc[2 * j + 1] += d * bb.y + a * ee.y;
      }
    }
    const i64 gr = r0 + r;
    if (gr < M) {
      const u64* Cl = C + l * sC + gr * N;
      u64* Zl = Z + l * sZ + gr * N;
#pragma unroll
      for (int j = 0; j < NT; ++j)
        if (j < N) Zl[j] = (Cl[j] + acc[j]) & msk;
    }
  }
}

namespace {
template <int L>
int launch_thin(i64 batch, cudaStream_t s, uint64_t* Z, int64_t sZ, int64_t bZ, const uint64_t* C, int64_t sC,
                int64_t bC, const SimOperand& X, const uint64_t* A, int64_t sA, int64_t bA, const SimOperand& Y,
                const uint64_t* B, int64_t sB, int64_t bB, int M, int K, int N, int p0, int width) {
  if (K <= 32 && N <= 32 && M >= 4096) {
    const int KP = K | 1;
    const int nt = N <= 16 ? 16 : (N <= 20 ? 20 : 32);
    const size_t smem = 8 * ((size_t)(L + 1) * K * nt + (size_t)(L + 1) * TALL_R * KP);
    const int groups = (M + TALL_R - 1) / TALL_R;
    const unsigned g = (unsigned)min((i64)groups, (i64)dev_sms() * 16);
    dim3 grid(g, (unsigned)batch);
#define TALL_CASE(NT_)                                                                                         \
  {                                                                                                            \
    static bool attr = false;                                                                                  \
    if (!attr) {                                                                                               \
      if (cudaFuncSetAttribute(k_beaver_tall<L, NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024) != \
          cudaSuccess)                                                                                         \
        return MPX_ERR_CUDA;                                                                                   \
      attr = true;                                                                                             \
    }                                                                                                          \
    k_beaver_tall<L, NT_><<<grid, 32 * L, smem, s>>>(Z, sZ, bZ, C, sC, bC, X, A, sA, bA, Y, B, sB, bB, M, K, N, \
                                                      p0, ring_mask(width));                                    \
  }
    if (nt == 16) TALL_CASE(16) else if (nt == 20) TALL_CASE(20) else TALL_CASE(32)
#undef TALL_CASE
    return launch_status();
  }
  return MPX_ERR_ARG;
}

// shapes the thin kernels take (MPX_THIN=0 disables them for A/B runs)
bool thin_fits(int L, i64 M, i64 K, i64 N, int width) {
  if (const char* e = getenv("MPX_THIN"))
    if (atoi(e) == 0) return false;
  return K <= 32 && N <= 32 && M >= 4096;
}
}  // namespace

extern "C" int mpx_beaver_gemm_sim(uint64_t* Z, int64_t sZ, int64_t bZ, const uint64_t* C, int64_t sC, int64_t bC,
                                   const uint64_t* X, int64_t x_ps, int64_t x_sr, int64_t x_sc, int64_t x_js,
                                   const uint64_t* A, int64_t sA, int64_t bA, const uint64_t* Y, int64_t y_ps,
                                   int64_t y_sr, int64_t y_sc, int64_t y_js, const uint64_t* B, int64_t sB,
                                   int64_t bB, int L, int64_t batch, int64_t M, int64_t K, int64_t N, int p0,
                                   int width, void* stream) {
  CHECK_ARG(Z && C && X && A && Y && B && M >= 1 && K >= 1 && N >= 1 && width >= 1 && width <= 64);
  CHECK_ARG(L >= 2 && L <= 4 && p0 < L && batch >= 1);
  CHECK_ARG(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31) && M * K < (1ll << 40) && K * N < (1ll << 40));
  // least padded output area; on a tie the larger tile, unless the product
  // is too small to fill the SMs (small outputs: the split-K grid is
  // tiles x at most K / 16 chunks), where more, smaller tiles spread the
  // per-CTA reduction over more SMs (LeNet fc2: 128 x 500 x 10 on 32 vs 124 CTAs)
  const bool small = (M * N * batch) / 1024 * max((i64)1, K / (2 * BS_BK)) < (i64)dev_sms() * 4;
  int best = 0;
  i64 best_cost = -1, best_area = 0;
  for (int c = 0; c < kNumSimCfgs; ++c) {
    const i64 bm = kSimCfgs[c].bm, bn = kSimCfgs[c].bn;
    const i64 cost = ((M + bm - 1) / bm) * bm * ((N + bn - 1) / bn) * bn;
    const bool tie_better = small ? bm * bn < best_area : bm * bn > best_area;
    if (best_cost < 0 || cost < best_cost || (cost == best_cost && tie_better)) {
      best = c;
      best_cost = cost;
      best_area = bm * bn;
    }
  }
  if (const char* e = getenv("MPX_BS_CFG")) best = min(max(atoi(e), 0), kNumSimCfgs - 1);  // sweeps
  const SimOperand xo{X, x_ps, x_sr, x_sc, x_js}, yo{Y, y_ps, y_sr, y_sc, y_js};
  cudaStream_t s = (cudaStream_t)stream;
  if (thin_fits(L, M, K, N, width) && batch <= 65535) {
    if (L == 2)
      return launch_thin<2>(batch, s, Z, sZ, bZ, C, sC, bC, xo, A, sA, bA, yo, B, sB, bB, (int)M, (int)K, (int)N, p0,
                            width);
    if (L == 3)
      return launch_thin<3>(batch, s, Z, sZ, bZ, C, sC, bC, xo, A, sA, bA, yo, B, sB, bB, (int)M, (int)K, (int)N, p0,
                            width);
    return launch_thin<4>(batch, s, Z, sZ, bZ, C, sC, bC, xo, A, sA, bA, yo, B, sB, bB, (int)M, (int)K, (int)N, p0,
                          width);
  }
  if (L == 2)
    return dispatch_sim<2>(best, K, batch, s, Z, sZ, bZ, C, sC, bC, xo, A, sA, bA, yo, B, sB, bB, (int)M, (int)N, p0,
                           width);
  if (L == 3)
    return dispatch_sim<3>(best, K, batch, s, Z, sZ, bZ, C, sC, bC, xo, A, sA, bA, yo, B, sB, bB, (int)M, (int)N, p0,
                           width);
  return dispatch_sim<4>(best, K, batch, s, Z, sZ, bZ, C, sC, bC, xo, A, sA, bA, yo, B, sB, bB, (int)M, (int)N, p0,
                         width);
}
