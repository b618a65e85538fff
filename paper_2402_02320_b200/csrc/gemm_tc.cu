// Z_2^64 GEMM on the 5th-gen tensor cores (tcgen05, kind::i8, TMEM, TMA).
//
// A 64-bit ring product is exact from 8-bit limbs: with A = sum_i 2^(8i) A_i,
// B = sum_j 2^(8j) B_j (u8 limb planes),
//     A @ B mod 2^64 = sum_{d=0..7} 2^(8d) * sum_{i+j=d} A_i @ B_j   (mod 2^64)
// i.e. 36 u8 x u8 -> s32 limb products, accumulated per diagonal d in its own
// TMEM accumulator. Diagonal d only matters mod 2^(64-8d): d >= 4 needs 32
// bits (wrap-around harmless), d <= 3 stays below 2^32 while K <= 16384
// ((d+1) * K * 255^2 < 2^32), so the u32 reading of each s32 accumulator
// recombines exactly (SURVEY §7 hard part 1, checked on all-0xFF inputs in
// tests/test_gemm_tc.py).
//
// CTA tile 128 (M) x 64 (N): 8 accumulators x 64 columns = all 512 TMEM
// columns. Per k-block of 128 bytes: all 8 B-limb tiles stay resident (double
// buffered) while the 8 A-limb tiles stream through a 4-stage ring; A_i meets
// B_0..B_{7-i}. Warp roles: w0 TMA producer, w1 MMA issuer (+TMEM owner),
// w2..w5 epilogue (TMEM -> registers -> limb recombination -> global).
// Operand tiles are TMA-loaded with 128-byte swizzle; UMMA smem descriptors
// are K-major SWIZZLE_128B.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"

#define TC_BM 128
#define TC_BK 128
#define TC_A_TILE (TC_BM * TC_BK)          // 16 KB
#define TC_GROUP_M 16
// Two instantiations: "wide" (N tile 64, all 512 TMEM columns, 1 CTA/SM,
// deep rings) for long reductions; "narrow" (N tile 32, 256 columns, short
// rings) fits 2 CTAs per SM so one CTA's epilogue overlaps the other's
// mainloop - the shape of short-K / many-tile products (conv backward, thin
// layers), where the epilogue is a large share of each tile.
constexpr int tc_smem_bytes(int bn, int ast, int bst) { return ast * TC_A_TILE + bst * 8 * bn * TC_BK + 1024 + 256; }
#define TC_WIDE 64, 6, 2
#define TC_NARROW 32, 4, 1

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z), "r"(z), "r"(z), "r"(z));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// K-major, 128-byte swizzle UMMA shared-memory descriptor (version 1 = sm100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

#define TMEM_LD32(taddr, v)                                                                              \
  asm volatile(                                                                                          \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"   \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                        \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),        \
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),      \
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),      \
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                           \
      : "r"(taddr))

struct TcArgs {
  u64* C;
  const u64* Cin;  // optional addend (C = Cin + A@B), same ldc as C
  i64 sCin;
  i64 ldc;
  i64 sC;        // batch stride of C (elements)
  int M, N;      // true output extent
  int Mpad, Npad;
  int nk;        // k-blocks of TC_BK bytes per CTA (split-K slice)
  int nk_total;  // k-blocks of the whole reduction
  int ksplit;    // CTAs per output tile along K; > 1 => wrapping atomic adds
  int accumulate;
  u64 msk;
};

template <int BN, int AST, int BST>
__global__ void __launch_bounds__(192, BN == 32 ? 2 : 1)
    k_gemm_limbs_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    TcArgs args) {
  constexpr int B_TILE = BN * TC_BK;
  constexpr int B_STAGE = 8 * B_TILE;
  constexpr uint32_t TMEM_COLS = 8 * BN;  // one accumulator per diagonal
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + AST * TC_A_TILE;
  uint64_t* bars = (uint64_t*)(sB + BST * B_STAGE);
  uint64_t* fullA = bars;
  uint64_t* emptyA = bars + AST;
  uint64_t* fullB = bars + 2 * AST;
  uint64_t* emptyB = bars + 2 * AST + BST;
  uint64_t* tmem_full = bars + 2 * AST + 2 * BST;
  uint32_t* tmem_holder = (uint32_t*)(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // grouped rasterization: consecutive CTAs walk TC_GROUP_M row tiles of one
  // column band, so a wave shares both A and B k-slabs through L2
  const int tiles_m = args.Mpad / TC_BM, tiles_n = args.Npad / BN;
  const int ks = blockIdx.x % args.ksplit;            // split-K slice of this CTA
  const int lin = blockIdx.x / args.ksplit;
  const int kb0 = ks * args.nk;
  const int nk = min(args.nk, args.nk_total - kb0);
  const int per_group = TC_GROUP_M * tiles_n;
  const int g = lin / per_group;
  const int first_m = g * TC_GROUP_M;
  const int gm = min(TC_GROUP_M, tiles_m - first_m);
  const int in_g = lin - g * per_group;
  const int m0 = (first_m + in_g % gm) * TC_BM;
  const int n0 = (in_g / gm) * BN;
  const int z = blockIdx.z;

  if (threadIdx.x == 0) {
    for (int s = 0; s < AST; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < BST; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int as = 0;
      uint32_t aph = 0;
      for (int kb = 0; kb < nk; ++kb) {
        const int bs = kb % BST;
        const uint32_t bph = (uint32_t)((kb / BST) & 1);
        mbar_wait(&emptyB[bs], bph ^ 1);
        mbar_expect_tx(&fullB[bs], B_STAGE);
        for (int j = 0; j < 8; ++j)
          tma_load_2d(sB + bs * B_STAGE + j * B_TILE, &mapB, &fullB[bs], (kb0 + kb) * TC_BK,
                      (z * 8 + j) * args.Npad + n0);
        for (int i = 0; i < 8; ++i) {
          mbar_wait(&emptyA[as], aph ^ 1);
          mbar_expect_tx(&fullA[as], TC_A_TILE);
          tma_load_2d(sA + as * TC_A_TILE, &mapA, &fullA[as], (kb0 + kb) * TC_BK, (z * 8 + i) * args.Mpad + m0);
          if (++as == AST) {
            as = 0;
            aph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      // Descriptors are precomputed: the start address is the low field, so
      // advancing within shared memory is a plain add of (bytes >> 4).
      const uint32_t idesc = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
      const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA));
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sB));
      int as = 0;
      uint32_t aph = 0;
      for (int kb = 0; kb < nk; ++kb) {
        const int bs = kb % BST;
        const uint32_t bph = (uint32_t)((kb / BST) & 1);
        mbar_wait(&fullB[bs], bph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t bd0 = b_desc0 + (uint64_t)((bs * B_STAGE) >> 4);
        const uint32_t first = kb == 0 ? 0u : 1u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          mbar_wait(&fullA[as], aph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = a_desc0 + (uint64_t)((as * TC_A_TILE) >> 4);
#pragma unroll
          for (int j = 0; j <= 7 - i; ++j) {
            const uint32_t d_tmem = tmem_base + (uint32_t)((i + j) * BN);
            const uint64_t bd = bd0 + (uint64_t)((j * B_TILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < TC_BK / 32; ++kk)
              mma_i8(d_tmem, ad + 2 * kk, bd + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : first);
          }
          umma_commit(&emptyA[as]);  // slot free once these MMAs retire
          if (++as == AST) {
            as = 0;
            aph ^= 1;
          }
        }
        umma_commit(&emptyB[bs]);
      }
      umma_commit(tmem_full);
    }
  } else {
    // ---------------- epilogue: warps 2..5 ----------------
    // TMEM lane = tile row, so a thread holds one row. Narrow (short-K)
    // tiles transpose each 32x32 u64 block through shared memory (the
    // operand ring is idle once tmem_full fires) so global loads/stores run
    // along rows, 256 B per warp instruction.
    const int sp = warp & 3;  // TMEM sub-partition this warp may access
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    u64* stage = reinterpret_cast<u64*>(smem) + sp * (32 * 33);
    const i64 rbase = (i64)m0 + sp * 32;
    u64* Cz = args.C + (i64)z * args.sC;
    const u64* Cin = args.Cin ? args.Cin + (i64)z * args.sCin : nullptr;
    for (int c = 0; c < BN / 32; ++c) {
      u64 res[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) res[t] = 0;
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        uint32_t v[32];
        const uint32_t taddr = tmem_base + ((uint32_t)(sp * 32) << 16) + (uint32_t)(d * BN + c * 32);
        TMEM_LD32(taddr, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int t = 0; t < 32; ++t) res[t] += (u64)v[t] << (8 * d);
      }
      if constexpr (BN == 64) {
        // wide / long-K tiles: per-row direct stores (measured 4.17 vs 4.91 ms
        // staged at 4096^2 x 8192; the epilogue is a small share there)
        const i64 row = rbase + lane;
        if (row < args.M) {
          u64* Crow = Cz + row * args.ldc;
          const u64* Cinr = Cin ? Cin + row * args.ldc : nullptr;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int col = n0 + c * 32 + t;
            if (col < args.N) {
              if (args.ksplit > 1) {
                atomicAdd(reinterpret_cast<unsigned long long*>(Crow + col), (unsigned long long)res[t]);
              } else {
                u64 v = res[t];
                if (Cinr) v += Cinr[col];
                else if (args.accumulate) v += Crow[col];
                Crow[col] = v & args.msk;
              }
            }
          }
        }
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t) stage[lane * 33 + t] = res[t];
        __syncwarp();
        const int col = n0 + c * 32 + lane;
        const int rmax = (col < args.N) ? (int)min((i64)32, (i64)args.M - rbase) : 0;
        u64* dst = Cz + rbase * args.ldc + col;
        const u64* src = Cin ? Cin + rbase * args.ldc + col : (args.accumulate ? dst : nullptr);
        if (args.ksplit > 1) src = nullptr;
        // 8 addend loads in flight before the stores that use them
        for (int h = 0; h < 32; h += 8) {
          u64 add[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) add[r] = (src && h + r < rmax) ? src[(i64)(h + r) * args.ldc] : 0ull;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            if (h + r < rmax) {
              const u64 val = stage[(h + r) * 33 + lane];
              if (args.ksplit > 1)
                atomicAdd(reinterpret_cast<unsigned long long*>(dst + (i64)(h + r) * args.ldc),
                          (unsigned long long)val);
              else
                dst[(i64)(h + r) * args.ldc] = (val + add[r]) & args.msk;
            }
          }
        }
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// --------------------------------------------------------------------------
// Persistent variant for short reductions with large outputs (conv backward
// dX: K of one or two k-blocks, M x N in the 10^7-10^8 range). One CTA per SM
// walks 128 x 64 output tiles blockIdx.x, +gridDim.x, ... The 8 diagonal
// accumulators take all 512 TMEM columns, so instead of double-buffering TMEM
// the epilogue drains them into shared memory right away and hands TMEM back
// (tmem_empty) before its slow part — the C-addend loads and the coalesced
// global stores — which then overlaps the next tile's TMA loads and MMAs.
#define TCP_BN 64
#define TCP_AST 4
#define TCP_BST 1
#define TCP_STAGE_BYTES (4 * 2 * 32 * 33 * 8)
constexpr int tcp_smem_bytes() {
  return TCP_AST * TC_A_TILE + TCP_BST * 8 * TCP_BN * TC_BK + TCP_STAGE_BYTES + 1024 + 256;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(192, 1)
    k_gemm_limbs_tc_pers(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                         TcArgs args, int batch) {
  constexpr int BN = TCP_BN, AST = TCP_AST, BST = TCP_BST;
  constexpr int B_TILE = BN * TC_BK;
  constexpr int B_STAGE = 8 * B_TILE;
  constexpr uint32_t ACC_COLS = 8 * BN;  // 8 diagonals = all 512 columns
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + AST * TC_A_TILE;
  u64* stage_all = reinterpret_cast<u64*>(sB + BST * B_STAGE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stage_all) + TCP_STAGE_BYTES);
  uint64_t* fullA = bars;
  uint64_t* emptyA = bars + AST;
  uint64_t* fullB = bars + 2 * AST;
  uint64_t* emptyB = bars + 2 * AST + BST;
  uint64_t* tfull = bars + 2 * AST + 2 * BST;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = (uint32_t*)(tempty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_m = args.Mpad / TC_BM, tiles_n = args.Npad / BN;
  const int per_batch = tiles_m * tiles_n;
  const int total = per_batch * batch;
  const int nk = args.nk_total;

  if (threadIdx.x == 0) {
    for (int s = 0; s < AST; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < BST; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);  // one arrival per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(ACC_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  auto tile_coords = [&](int t, int& z, int& m0, int& n0) {
    z = t / per_batch;
    const int lin = t - z * per_batch;
    const int per_group = TC_GROUP_M * tiles_n;
    const int g = lin / per_group;
    const int first_m = g * TC_GROUP_M;
    const int gm = min(TC_GROUP_M, tiles_m - first_m);
    const int in_g = lin - g * per_group;
    m0 = (first_m + in_g % gm) * TC_BM;
    n0 = (in_g / gm) * BN;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int as = 0, gkb = 0;
      uint32_t aph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int z, m0, n0;
        tile_coords(t, z, m0, n0);
        for (int kb = 0; kb < nk; ++kb, ++gkb) {
          const int bs = gkb % BST;
          const uint32_t bph = (uint32_t)((gkb / BST) & 1);
          mbar_wait(&emptyB[bs], bph ^ 1);
          mbar_expect_tx(&fullB[bs], B_STAGE);
          for (int j = 0; j < 8; ++j)
            tma_load_2d(sB + bs * B_STAGE + j * B_TILE, &mapB, &fullB[bs], kb * TC_BK, (z * 8 + j) * args.Npad + n0);
          for (int i = 0; i < 8; ++i) {
            mbar_wait(&emptyA[as], aph ^ 1);
            mbar_expect_tx(&fullA[as], TC_A_TILE);
            tma_load_2d(sA + as * TC_A_TILE, &mapA, &fullA[as], kb * TC_BK, (z * 8 + i) * args.Mpad + m0);
            if (++as == AST) {
              as = 0;
              aph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
      const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA));
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sB));
      int as = 0, gkb = 0, it = 0;
      uint32_t aph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        mbar_wait(tempty, (uint32_t)((it & 1) ^ 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < nk; ++kb, ++gkb) {
          const int bs = gkb % BST;
          const uint32_t bph = (uint32_t)((gkb / BST) & 1);
          mbar_wait(&fullB[bs], bph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t bd0 = b_desc0 + (uint64_t)((bs * B_STAGE) >> 4);
          const uint32_t first = kb == 0 ? 0u : 1u;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            mbar_wait(&fullA[as], aph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t ad = a_desc0 + (uint64_t)((as * TC_A_TILE) >> 4);
#pragma unroll
            for (int j = 0; j <= 7 - i; ++j) {
              const uint32_t d_tmem = tmem_base + (uint32_t)((i + j) * BN);
              const uint64_t bd = bd0 + (uint64_t)((j * B_TILE) >> 4);
#pragma unroll
              for (int kk = 0; kk < TC_BK / 32; ++kk)
                mma_i8(d_tmem, ad + 2 * kk, bd + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : first);
            }
            umma_commit(&emptyA[as]);
            if (++as == AST) {
              as = 0;
              aph ^= 1;
            }
          }
          umma_commit(&emptyB[bs]);
        }
        umma_commit(tfull);
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 ----------------
    const int sp = warp & 3;
    u64* stage = stage_all + sp * (2 * 32 * 33);
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      int z, m0, n0;
      tile_coords(t, z, m0, n0);
      mbar_wait(tfull, (uint32_t)(it & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        u64 res[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) res[q] = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          uint32_t v[32];
          const uint32_t taddr = tmem_base + ((uint32_t)(sp * 32) << 16) + (uint32_t)(d * BN + c * 32);
          TMEM_LD32(taddr, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 32; ++q) res[q] += (u64)v[q] << (8 * d);
        }
#pragma unroll
        for (int q = 0; q < 32; ++q) stage[c * 32 * 33 + lane * 33 + q] = res[q];
      }
      // accumulators drained: the MMA warp may start the next tile
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      const i64 rbase = (i64)m0 + sp * 32;
      const i64 rows = min((i64)32, (i64)args.M - rbase);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int col = n0 + c * 32 + lane;
        const int rmax = (col < args.N) ? (int)rows : 0;
        u64* dst = args.C + (i64)z * args.sC + rbase * args.ldc + col;
        const u64* src = args.Cin ? args.Cin + (i64)z * args.sCin + rbase * args.ldc + col
                                  : (args.accumulate ? dst : nullptr);
        const u64* st = stage + c * 32 * 33;
        for (int h = 0; h < 32; h += 16) {
          u64 add[16];
#pragma unroll
          for (int r = 0; r < 16; ++r) add[r] = (src && h + r < rmax) ? src[(i64)(h + r) * args.ldc] : 0ull;
#pragma unroll
          for (int r = 0; r < 16; ++r)
            if (h + r < rmax) dst[(i64)(h + r) * args.ldc] = (st[(h + r) * 33 + lane] + add[r]) & args.msk;
        }
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ACC_COLS));
  }
}

// --------------------------------------------------------------------------
// Limb split: u64 matrix -> 8 u8 planes. `trans` = 0: plane[i][r][coff + c];
// trans = 1: plane[i][c][coff + r] (K-major operand from a row-major KxN).

__device__ __forceinline__ void bytes_transpose8(const u64 (&w)[8], u64 (&p)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    u64 v = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) v |= ((w[c] >> (8 * i)) & 0xFFull) << (8 * c);
    p[i] = v;
  }
}

// non-transposed: each thread takes 8 consecutive columns of one row
__global__ void k_limb_split(uint8_t* __restrict__ out, const u64* __restrict__ A, i64 rows, i64 cols, i64 lda,
                             i64 plane, i64 pitch, i64 coff) {
  const i64 groups_per_row = (cols + 7) / 8;
  const i64 total = rows * groups_per_row;
  GRID_STRIDE(t, total) {
    const i64 r = t / groups_per_row;
    const i64 c0 = (t - r * groups_per_row) * 8;
    u64 w[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) w[c] = (c0 + c < cols) ? A[r * lda + c0 + c] : 0ull;
    u64 p[8];
    bytes_transpose8(w, p);
    uint8_t* dst = out + r * pitch + coff + c0;
    if (c0 + 8 <= cols && (((uintptr_t)dst) & 7) == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<u64*>(dst + i * plane) = p[i];
    } else {
      for (int i = 0; i < 8; ++i)
        for (int c = 0; c < 8 && c0 + c < cols; ++c) dst[i * plane + c] = (uint8_t)(p[i] >> (8 * c));
    }
  }
}

// transposed via a 64 (k) x 32 (n) smem tile
__global__ void __launch_bounds__(256) k_limb_split_t(uint8_t* __restrict__ out, const u64* __restrict__ A,
                                                      i64 rows, i64 cols, i64 lda, i64 plane, i64 pitch,
                                                      i64 coff) {
  __shared__ u64 tile[64][33];
  const i64 k0 = (i64)blockIdx.y * 64;
  const i64 n0 = (i64)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int kk = ty; kk < 64; kk += 8) {
    const i64 k = k0 + kk, n = n0 + tx;
    tile[kk][tx] = (k < rows && n < cols) ? A[k * lda + n] : 0ull;
  }
  __syncthreads();
  // 8 lanes cover one output row's 64 contiguous k-bytes (two full sectors)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = warp * 4 + (lane >> 3);
  const int g = lane & 7;
  const i64 gn = n0 + n;
  const i64 gk = k0 + g * 8;
  if (gn < cols && gk < rows) {
    u64 w[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) w[c] = tile[g * 8 + c][n];
    u64 p[8];
    bytes_transpose8(w, p);
    uint8_t* dst = out + gn * pitch + coff + gk;
    if (gk + 8 <= rows && (((uintptr_t)dst) & 7) == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<u64*>(dst + i * plane) = p[i];
    } else {
      for (int i = 0; i < 8; ++i)
        for (int c = 0; c < 8 && gk + c < rows; ++c) dst[i * plane + c] = (uint8_t)(p[i] >> (8 * c));
    }
  }
}

extern "C" int mpx_limb_split(uint8_t* out, const uint64_t* A, int64_t rows, int64_t cols, int64_t lda,
                              int64_t plane, int64_t pitch, int64_t coff, int trans, void* stream) {
  CHECK_ARG(out && A && rows >= 0 && cols >= 0 && lda >= cols);
  if (rows == 0 || cols == 0) return MPX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (!trans) {
    k_limb_split<<<grid_for(rows * ((cols + 7) / 8)), MPX_THREADS, 0, s>>>(out, A, rows, cols, lda, plane,
                                                                           pitch, coff);
  } else {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 63) / 64));
    CHECK_ARG(grid.y <= 65535);
    k_limb_split_t<<<grid, 256, 0, s>>>(out, A, rows, cols, lda, plane, pitch, coff);
  }
  return launch_status();
}

// --------------------------------------------------------------------------
// Beaver operand preparation (basic.py:72-75 as one K-concatenated GEMM per
// party): A8[l] = limbs of [D | A_l] (M x 2K), B8[l] = limbs of
// [B_l + [l==p0] E ; E]^T (N x 2K, K-major). One launch per side for all
// parties; D and E are read once per party slice.

__global__ void k_beaver_limbs_a(uint8_t* __restrict__ A8, const u64* __restrict__ D, const u64* __restrict__ A,
                                 i64 a_ps, int L, i64 M, i64 Kd, i64 Mpad, i64 Kpad) {
  const i64 gpr = Kpad / 8;  // 8-column groups per row (columns >= 2K are zero padding)
  const i64 total = (i64)L * M * gpr;
  GRID_STRIDE(t, total) {
    const i64 g = t % gpr;
    const i64 rl = t / gpr;
    const i64 r = rl % M, l = rl / M;
    const i64 c0 = g * 8;
    u64 w[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const i64 cc = c0 + c;
      w[c] = cc < Kd ? D[r * Kd + cc] : (cc < 2 * Kd ? A[l * a_ps + r * Kd + (cc - Kd)] : 0ull);
    }
    u64 pl[8];
    bytes_transpose8(w, pl);
    uint8_t* dst = A8 + (l * 8) * Mpad * Kpad + r * Kpad + c0;
    const i64 plane = Mpad * Kpad;
    if (c0 + 8 <= Kpad && (((uintptr_t)dst) & 7) == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<u64*>(dst + i * plane) = pl[i];
    } else {
      for (int i = 0; i < 8; ++i)
        for (int c = 0; c < 8 && c0 + c < Kpad; ++c) dst[i * plane + c] = (uint8_t)(pl[i] >> (8 * c));
    }
  }
}

// transposed side through a 64 (k) x 32 (n) smem tile; blockIdx.z = party
__global__ void __launch_bounds__(256) k_beaver_limbs_b(uint8_t* __restrict__ B8, const u64* __restrict__ Bm,
                                                        i64 b_ps, const u64* __restrict__ E, int p0, i64 Kd, i64 N,
                                                        i64 Npad, i64 Kpad) {
  __shared__ u64 tile[64][33];
  const int l = blockIdx.z;
  const i64 k0 = (i64)blockIdx.y * 64;  // over the concatenated 2K rows
  const i64 n0 = (i64)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int kk = ty; kk < 64; kk += 8) {
    const i64 k = k0 + kk, n = n0 + tx;
    u64 v = 0;
    if (n < N) {
      if (k < Kd) {
        v = Bm[l * b_ps + k * N + n];
        if (l == p0) v += E[k * N + n];
      } else if (k < 2 * Kd) {
        v = E[(k - Kd) * N + n];
      }
    }
    tile[kk][tx] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = warp * 4 + (lane >> 3);
  const int g = lane & 7;
  const i64 gn = n0 + n, gk = k0 + g * 8;
  if (gn < Npad && gk < Kpad) {
    u64 w[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) w[c] = tile[g * 8 + c][n];
    u64 pl[8];
    bytes_transpose8(w, pl);
    uint8_t* dst = B8 + ((i64)l * 8) * Npad * Kpad + gn * Kpad + gk;
    const i64 plane = Npad * Kpad;
#pragma unroll
    for (int i = 0; i < 8; ++i) *reinterpret_cast<u64*>(dst + i * plane) = pl[i];
  }
}

extern "C" int mpx_beaver_limbs(uint8_t* A8, uint8_t* B8, const uint64_t* D, const uint64_t* E, const uint64_t* A,
                                int64_t a_ps, const uint64_t* B, int64_t b_ps, int L, int64_t M, int64_t K,
                                int64_t N, int64_t Mpad, int64_t Npad, int64_t Kpad, int p0, void* stream) {
  CHECK_ARG(A8 && B8 && D && E && A && B && L >= 1 && L <= 65535 && M >= 1 && K >= 1 && N >= 1);
  CHECK_ARG(Mpad >= M && Npad >= N && Kpad >= 2 * K && Kpad % 64 == 0 && Kpad % 8 == 0);
  cudaStream_t s = (cudaStream_t)stream;
  const i64 ta = (i64)L * M * ((Kpad + 7) / 8);
  // A side also zero-fills the K padding columns (groups beyond 2K read as 0)
  k_beaver_limbs_a<<<grid_for(ta), MPX_THREADS, 0, s>>>(A8, D, A, a_ps, L, M, K, Mpad, Kpad);
  dim3 grid((unsigned)((Npad + 31) / 32), (unsigned)(Kpad / 64), (unsigned)L);
  CHECK_ARG(grid.y <= 65535);
  k_beaver_limbs_b<<<grid, 256, 0, s>>>(B8, B, b_ps, E, p0, K, N, Npad, Kpad);
  return launch_status();
}

// --------------------------------------------------------------------------
// Host: tensor maps + launch

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

static int make_map(CUtensorMap* map, const uint8_t* base, i64 rows, i64 kbytes, int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return MPX_ERR_CUDA;
  cuuint64_t dims[2] = {(cuuint64_t)kbytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kbytes};
  cuuint32_t box[2] = {TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? MPX_OK : MPX_ERR_CUDA;
}

// C[z] (+)= sum_{i+j<=7} 2^(8(i+j)) A8[z][i] @ B8[z][j]^T  (mod 2^width)
// A8: [batch][8][Mpad][Kpad] u8, B8: [batch][8][Npad][Kpad] u8, zero padded;
// Mpad % 128 == 0, Npad % 64 == 0, Kpad % 128 == 0, Kpad <= 16384.
extern "C" int mpx_gemm_limbs(uint64_t* C, const uint8_t* A8, const uint8_t* B8, int64_t batch, int64_t M,
                              int64_t N, int64_t Mpad, int64_t Npad, int64_t Kpad, int64_t ldc, int64_t sC,
                              int accumulate, int width, int ksplit, const uint64_t* Cin, int64_t sCin,
                              void* stream) {
  CHECK_ARG(C && A8 && B8 && batch >= 1 && batch <= 65535 && M >= 1 && N >= 1 && width >= 1 && width <= 64);
  CHECK_ARG(Mpad % TC_BM == 0 && Npad % 32 == 0 && Kpad % TC_BK == 0 && Kpad >= TC_BK);
  const int nk_total = (int)(Kpad / TC_BK);
  if (ksplit < 1) ksplit = 1;
  if (ksplit > nk_total) ksplit = nk_total;
  int nk_per = (nk_total + ksplit - 1) / ksplit;
  ksplit = (nk_total + nk_per - 1) / nk_per;
  // exactness: each CTA's s32 diagonal accumulators see at most 16384 of K
  CHECK_ARG((i64)nk_per * TC_BK <= 16384);
  // split-K adds partials with wrapping 64-bit atomics: exact mod 2^64 only
  CHECK_ARG(ksplit == 1 || width == 64);
  CHECK_ARG(!(Cin && accumulate));
  if (ksplit > 1 && Cin) {
    // partial sums land on a copy of the addend
    for (i64 z = 0; z < batch; ++z)
      if (cudaMemcpy2DAsync(C + z * sC, (size_t)ldc * 8, Cin + z * sCin, (size_t)ldc * 8, (size_t)N * 8,
                            (size_t)M, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) != cudaSuccess)
        return MPX_ERR_CUDA;
    Cin = nullptr;
  } else if (ksplit > 1 && !accumulate) {
    for (i64 z = 0; z < batch; ++z)
      if (cudaMemset2DAsync(C + z * sC, (size_t)ldc * 8, 0, (size_t)N * 8, (size_t)M, (cudaStream_t)stream) !=
          cudaSuccess)
        return MPX_ERR_CUDA;
  }
  CHECK_ARG(M <= Mpad && N <= Npad && ldc >= N);
  CHECK_ARG(batch * 8 * Mpad < (1ll << 31) && batch * 8 * Npad < (1ll << 31));
  CUtensorMap mapA, mapB;
  if (make_map(&mapA, A8, batch * 8 * Mpad, Kpad, TC_BM) != MPX_OK) return MPX_ERR_CUDA;
  // persistent 128x64 tiles (epilogue overlapped with the next tile) for
  // short unsplit reductions over many output tiles; else narrow tiles when N
  // is not a multiple of 64 or the reduction is short, wide tiles otherwise
  const i64 ntiles64 = (Npad / 64) * (Mpad / TC_BM) * batch;
  // (one k-block per tile leaves too little MMA work to hide the epilogue:
  // measured slower there, faster at 2-4)
  const bool pers = Npad % 64 == 0 && ksplit == 1 && nk_total >= 2 && nk_total <= 4 && ntiles64 >= 4 * 148 &&
                    getenv("MPX_TC_NO_PERSIST") == nullptr;
  const bool narrow = !pers && ((Npad % 64 != 0) || nk_per <= 2);
  const int bn = narrow ? 32 : 64;
  if (make_map(&mapB, B8, batch * 8 * Npad, Kpad, bn) != MPX_OK) return MPX_ERR_CUDA;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(k_gemm_limbs_tc<TC_WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             tc_smem_bytes(TC_WIDE)) != cudaSuccess ||
        cudaFuncSetAttribute(k_gemm_limbs_tc<TC_NARROW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             tc_smem_bytes(TC_NARROW)) != cudaSuccess ||
        cudaFuncSetAttribute(k_gemm_limbs_tc_pers, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             tcp_smem_bytes()) != cudaSuccess)
      return MPX_ERR_CUDA;
    attr_set = true;
  }
  TcArgs a;
  a.C = C;
  a.Cin = Cin;
  a.sCin = sCin;
  a.ldc = ldc;
  a.sC = sC;
  a.M = (int)M;
  a.N = (int)N;
  a.Mpad = (int)Mpad;
  a.Npad = (int)Npad;
  a.nk = nk_per;
  a.nk_total = nk_total;
  a.ksplit = ksplit;
  a.accumulate = accumulate;
  a.msk = ring_mask(width);
  if (pers) {
    const unsigned g = (unsigned)min(ntiles64, (i64)148);
    k_gemm_limbs_tc_pers<<<g, 192, tcp_smem_bytes(), (cudaStream_t)stream>>>(mapA, mapB, a, (int)batch);
    return launch_status();
  }
  dim3 grid((unsigned)((Npad / bn) * (Mpad / TC_BM) * ksplit), 1, (unsigned)batch);
  if (narrow)
    k_gemm_limbs_tc<TC_NARROW><<<grid, 192, tc_smem_bytes(TC_NARROW), (cudaStream_t)stream>>>(mapA, mapB, a);
  else
    k_gemm_limbs_tc<TC_WIDE><<<grid, 192, tc_smem_bytes(TC_WIDE), (cudaStream_t)stream>>>(mapA, mapB, a);
  return launch_status();
}

int mpx_gemm_tc(uint64_t*, const uint64_t*, const uint64_t*, int64_t, int64_t, int64_t, int64_t, int64_t,
                int64_t, int64_t, int, int, cudaStream_t) {
  return MPX_ERR_UNSUPPORTED;  // the u64 entry point needs caller scratch: see mpx_gemm_limbs
}
