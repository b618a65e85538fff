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
// K-block-tiled limb planes: byte k of row r of a [Rpad][Kp] plane sits at
//   ((k / tw) * Rpad + r) * tw + (k % tw),   tw = min(128, Kp)
// so one TMA box (tw-wide k-block x 128 rows) is one contiguous 16 KB run of
// HBM instead of 128 row segments Kp bytes apart (measured: the TMA producer
// alone of an 8192 x 1024-byte operand ran at half the HBM bandwidth with
// row-major planes). Kp is 32, 64 or a multiple of 128 (kernels.kpad).
__host__ __device__ __forceinline__ int limb_tw(i64 Kp) { return Kp >= 128 ? 128 : (int)Kp; }
__host__ __device__ __forceinline__ i64 limb_off(i64 r, i64 k, i64 Rpad, int tw) {
  return ((k / tw) * Rpad + r) * tw + (k % tw);
}

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

// 3D box: consecutive limb planes land in consecutive 2D tiles of the stage
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
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
  int tw;       // limb-plane k-block tile width (bytes) and tiles per plane (per half if split)
  int nkt;
  int zl;       // split operands: parties per job (shared plane set = z / zl)
  i64 sCin_j;   // job stride of Cin (Cin of unit z at (z % zl) * sCin + (z / zl) * sCin_j)
  int dbg;      // timing experiments (MPX_TC_DBG bits): 1 one diagonal, 2 no stores, 4 no MMA, 8 no addend, 16 no drain
  int kb_half;  // > 0: split operands (persistent kernel only): k-blocks
                // [0, kb_half) pair shared A (mapA2) with party B (mapB),
                // the rest party A (mapA) with shared B (mapB2)
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
          tma_load_2d(sB + bs * B_STAGE + j * B_TILE, &mapB, &fullB[bs], 0,
                      ((z * 8 + j) * args.nkt + kb0 + kb) * args.Npad + n0);
        for (int i = 0; i < 8; ++i) {
          mbar_wait(&emptyA[as], aph ^ 1);
          mbar_expect_tx(&fullA[as], TC_A_TILE);
          tma_load_2d(sA + as * TC_A_TILE, &mapA, &fullA[as], 0, ((z * 8 + i) * args.nkt + kb0 + kb) * args.Mpad + m0);
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
// Persistent kernel: one CTA per SM walks work units u = blockIdx.x,
// +gridDim.x, ...; a unit is one 128 x 64 output tile and one slice of its
// k-blocks (split-K slices add their partials with wrapping 64-bit atomics,
// exact mod 2^64). The 8 diagonal accumulators take all 512 TMEM columns, so
// instead of double-buffering TMEM the epilogue drains them into registers
// (a thread owns one row: 64 u64) and hands TMEM back (tempty) before its
// global stores, which then overlap the next unit's TMA loads and MMAs.
// A ring of 4 single-limb stages + double-buffered B stages (8 limbs each)
// keep the tensor pipe fed across unit boundaries. N tiles of 64 also cover
// Npad % 64 == 32: the extra 32 B rows belong to the next plane (or are
// TMA zero-fill past the end) and only feed columns >= Npad, never stored.
// Template: BK = k-block bytes (128 / 64 / 32 with the matching 128B / 64B /
// 32B swizzle, so short reductions pad K to 32 or 64 instead of 128), BN =
// N tile (64, or 32 for outputs at most 32 wide: 256 TMEM columns).
#ifndef TCP_BST
#define TCP_BST 2
#endif
#define TCP_STAGE_TILE (32 * 33 * 8)  // one 32 x 32 u64 transpose tile per epilogue warp
#define TCP_STAGED_MAX_KB 4
// A ring: every byte of shared memory the B stages and the epilogue tiles
// leave (short-K products are load-latency bound: more A tiles in flight).
// MPX_TC_ARING_KB caps it at compile time for A/B runs (64 = the old ring).
#ifndef MPX_TC_ARING_KB
#define MPX_TC_ARING_KB 1024
#endif
// A limb tiles per TMA box / ring slot (one 3D box of AP consecutive limb
// planes); the B stage is one 3D box of all 8 limbs
#ifndef MPX_TC_AP
#define MPX_TC_AP 2
#endif
constexpr int tcp_fixed_bytes(int bk, int bn, bool staged, int ew) {
  return TCP_BST * 8 * bn * bk + (staged ? ew * TCP_STAGE_TILE : 0) + 1024 + 1024;
}
constexpr int tcp_ast_for(int bk, int bn, bool staged, int ew) {
  // limb tiles, rounded down to whole AP-tile ring slots
  return (((232448 - tcp_fixed_bytes(bk, bn, staged, ew)) / (TC_BM * bk)) < (MPX_TC_ARING_KB * 1024 / (TC_BM * bk))
              ? (232448 - tcp_fixed_bytes(bk, bn, staged, ew)) / (TC_BM * bk)
              : MPX_TC_ARING_KB * 1024 / (TC_BM * bk)) /
         MPX_TC_AP * MPX_TC_AP;
}
constexpr int tcp_smem_bytes(int bk, int bn, bool staged, int ew) {
  return tcp_ast_for(bk, bn, staged, ew) * TC_BM * bk + tcp_fixed_bytes(bk, bn, staged, ew);
}

// K-major UMMA shared-memory descriptor for a BK-byte-row swizzled tile
// (version 1 = sm100): SBO = 8 rows, layout 2 / 4 / 6 = 128B / 64B / 32B.
template <int BK>
__device__ __forceinline__ uint64_t umma_desc_sw(uint32_t saddr) {
  constexpr uint64_t layout = BK == 128 ? 2 : (BK == 64 ? 4 : 6);
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * BK) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= layout << 61;
  return d;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct TcpUnit {
  int z, m0, n0, kb0, nk, ks;
};

__device__ __forceinline__ TcpUnit tcp_unit(int u, const TcArgs& a, int tiles_m, int tiles_n, int bn) {
  TcpUnit t;
  t.ks = u % a.ksplit;
  const int lin_all = u / a.ksplit;
  const int per_batch = tiles_m * tiles_n;
  int lin;
  if (a.kb_half > 0) {
    // split operands: the parties of one job run the same tile back to back,
    // so the shared D / E limb blocks come from L2 for all but the first
    const int nz = a.zl;
    const int zi = lin_all % nz, rest = lin_all / nz;
    const int job = rest / per_batch;
    lin = rest - job * per_batch;
    t.z = job * nz + zi;
  } else {
    t.z = lin_all / per_batch;
    lin = lin_all - t.z * per_batch;
  }
  const int per_group = TC_GROUP_M * tiles_n;
  const int g = lin / per_group;
  const int first_m = g * TC_GROUP_M;
  const int gm = min(TC_GROUP_M, tiles_m - first_m);
  const int in_g = lin - g * per_group;
  t.m0 = (first_m + in_g % gm) * TC_BM;
  t.n0 = (in_g / gm) * bn;
  t.kb0 = t.ks * a.nk;
  t.nk = min(a.nk, a.nk_total - t.kb0);
  return t;
}

// EW = epilogue warps: 4 (one per TMEM lane quarter, all column chunks) or
// 8 (two per quarter, one 32-column chunk each: twice the TMEM drain and
// store parallelism for short reductions, where the epilogue paces a unit).
template <int BK, int BN, bool STAGED, int EW>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    k_gemm_limbs_tc_pers(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                         const __grid_constant__ CUtensorMap mapA2, const __grid_constant__ CUtensorMap mapB2,
                         TcArgs args, int batch) {
  constexpr int AST = tcp_ast_for(BK, BN, STAGED, EW) / MPX_TC_AP, BST = TCP_BST;  // AST: ring slots
  constexpr int AP = MPX_TC_AP;
  constexpr int A_TILE = TC_BM * BK;      // one limb tile; a ring slot holds AP of them
  constexpr int B_TILE = BN * BK;
  constexpr int B_STAGE = 8 * B_TILE;
  constexpr int NC = BN / 32;             // 32-column epilogue chunks
  constexpr uint32_t ACC_COLS = 8 * BN;  // 8 diagonals (512 or 256 columns)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + AST * AP * A_TILE;
  u64* stage_all = reinterpret_cast<u64*>(sB + BST * B_STAGE);
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stage_all) + (STAGED ? EW * TCP_STAGE_TILE : 0));
  uint64_t* fullA = bars;
  uint64_t* emptyA = bars + AST;
  uint64_t* fullB = bars + 2 * AST;
  uint64_t* emptyB = bars + 2 * AST + BST;
  uint64_t* tfull = bars + 2 * AST + 2 * BST;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = (uint32_t*)(tempty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_m = args.Mpad / TC_BM, tiles_n = (args.Npad + BN - 1) / BN;
  const int units = tiles_m * tiles_n * batch * args.ksplit;

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
    mbar_init(tempty, EW);  // one arrival per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
    if (args.kb_half > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA2) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB2) : "memory");
    }
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

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int as = 0, gkb = 0;
      uint32_t aph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const TcpUnit t = tcp_unit(u, args, tiles_m, tiles_n, BN);
        for (int kb = 0; kb < t.nk; ++kb, ++gkb) {
          const int bs = gkb % BST;
          const uint32_t bph = (uint32_t)((gkb / BST) & 1);
          const int kg = t.kb0 + kb;
          // split operands: first half = shared A x party B, second half =
          // party A x shared B (each half indexed from its own k origin)
          const bool lo = args.kb_half > 0 && kg < args.kb_half;
          const bool hi = args.kb_half > 0 && kg >= args.kb_half;
          const int kx = (hi ? kg - args.kb_half : kg) * BK;
          const CUtensorMap* mA = lo ? &mapA2 : &mapA;
          const CUtensorMap* mB = hi ? &mapB2 : &mapB;
          const int zs = args.kb_half > 0 ? t.z / args.zl : 0;
          const int zA = lo ? zs : t.z, zB = hi ? zs : t.z;
          mbar_wait(&emptyB[bs], bph ^ 1);
          mbar_expect_tx(&fullB[bs], B_STAGE);
          // all 8 B limb planes of the k-block in one 3D box
          tma_load_3d(sB + bs * B_STAGE, mB, &fullB[bs], kx % args.tw, (kx / args.tw) * args.Npad + t.n0, zB * 8);
          for (int i = 0; i < 8; i += AP) {
            mbar_wait(&emptyA[as], aph ^ 1);
            mbar_expect_tx(&fullA[as], AP * A_TILE);
            tma_load_3d(sA + as * AP * A_TILE, mA, &fullA[as], kx % args.tw, (kx / args.tw) * args.Mpad + t.m0,
                        zA * 8 + i);
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
      constexpr int MJ = 256 / BN;  // B limbs per MMA (N <= 256)
      const uint32_t idesc_base = (2u << 4) | ((uint32_t)(TC_BM >> 4) << 24);
      const uint64_t a_desc0 = umma_desc_sw<BK>(smem_u32(sA));
      const uint64_t b_desc0 = umma_desc_sw<BK>(smem_u32(sB));
      int as = 0, gkb = 0, it = 0;
      uint32_t aph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
        const TcpUnit t = tcp_unit(u, args, tiles_m, tiles_n, BN);
        mbar_wait(tempty, (uint32_t)((it & 1) ^ 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < t.nk; ++kb, ++gkb) {
          const int bs = gkb % BST;
          const uint32_t bph = (uint32_t)((gkb / BST) & 1);
          mbar_wait(&fullB[bs], bph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t bd0 = b_desc0 + (uint64_t)((bs * B_STAGE) >> 4);
          const uint32_t first = kb == 0 ? 0u : 1u;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i % AP == 0) {
              mbar_wait(&fullA[as], aph);  // limbs i .. i + AP - 1 landed
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            const uint64_t ad = a_desc0 + (uint64_t)(((as * AP + i % AP) * A_TILE) >> 4);
            // A_i meets B_0..B_{7-i}: the B limb tiles sit back to back in the
            // stage (rows of one K-major operand), and their diagonals i..7
            // are adjacent TMEM column blocks, so ONE MMA of N = nj * BN
            // covers nj limbs (N <= 256): 12 MMAs per k-step instead of 36
            // at BN = 64, 8 at BN = 32 (same tensor work, a third of the issue)
#pragma unroll
            for (int j0 = 0; j0 <= 7 - i; j0 += MJ) {
              const int nj = (8 - i - j0) < MJ ? (8 - i - j0) : MJ;
              const uint32_t d_tmem = tmem_base + (uint32_t)((i + j0) * BN);
              const uint64_t bd = bd0 + (uint64_t)((j0 * B_TILE) >> 4);
              const uint32_t id = idesc_base | ((uint32_t)((nj * BN) >> 3) << 17);
#pragma unroll
              for (int kk = 0; kk < BK / 32; ++kk)
                if (!(args.dbg & 4)) mma_i8(d_tmem, ad + 2 * kk, bd + 2 * kk, id, (i > 0 || kk > 0) ? 1u : first);
            }
            if (i % AP == AP - 1) {
              umma_commit(&emptyA[as]);  // slot free once these MMAs retire
              if (++as == AST) {
                as = 0;
                aph ^= 1;
              }
            }
          }
          umma_commit(&emptyB[bs]);
        }
        umma_commit(tfull);
      }
    }
  } else {
    // ---------------- epilogue: warps 2..(1 + EW) ----------------
    // TMEM lane = tile row: a thread owns one output row of the tile; with
    // 8 warps the second four take the second 32-column chunk.
    static_assert(EW == 4 || (EW == 8 && BN == 64 && STAGED), "8 epilogue warps: staged 64-wide tiles");
    const int sp = warp & 3;
    const int ew = warp - 2;
    constexpr int NCW = EW == 8 ? 1 : NC;  // chunks per warp
    const int c0 = EW == 8 ? (ew >> 2) : 0;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
      const TcpUnit t = tcp_unit(u, args, tiles_m, tiles_n, BN);
      const bool atom = args.ksplit > 1;
      const i64 rbase = (i64)t.m0 + sp * 32;
      const int rmax = (int)max((i64)0, min((i64)32, (i64)args.M - rbase));
      u64* Cz = args.C + (i64)t.z * args.sC + rbase * args.ldc;
      const u64* Cin =
          args.Cin ? args.Cin + (i64)(t.z % args.zl) * args.sCin + (i64)(t.z / args.zl) * args.sCin_j + rbase * args.ldc
                   : nullptr;
      // split slices meet in C through atomics (zeroed, or holding the
      // accumulate operand); slice 0 carries the Cin addend
      const u64* src = atom ? (t.ks == 0 ? Cin : nullptr) : (Cin ? Cin : (args.accumulate ? Cz : nullptr));
      u64* stage = stage_all + ew * (32 * 33);
      if constexpr (STAGED) {
        // the first chunk's addend block lands in the transpose tile
        // (cp.async, coalesced along the row) while the MMAs still run
        const int col = t.n0 + c0 * 32 + lane;
        const int rows = col < args.N ? rmax : 0;
#pragma unroll 8
        for (int r = 0; r < 32; ++r) {
          const u64* g = src + (i64)r * args.ldc + col;
          const uint32_t sz = (src && r < rows && !(args.dbg & 8)) ? 8u : 0u;  // 0: zero-fill
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(stage + r * 33 + lane)),
                       "l"(sz ? g : args.C), "r"(sz)
                       : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      mbar_wait(tfull, (uint32_t)(it & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // columns [32c, 32c + 32) of this warp's 32 rows, limb-recombined
      auto drain = [&](int c, u64 (&acc)[32]) {
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          if (((args.dbg & 1) && d > 0) || (args.dbg & 16)) break;  // timing experiments only (wrong results)
          uint32_t v[32];
          const uint32_t taddr = tmem_base + ((uint32_t)(sp * 32) << 16) + (uint32_t)(d * BN + c * 32);
          TMEM_LD32(taddr, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 32; ++q) acc[q] += (u64)v[q] << (8 * d);
        }
      };
      auto release = [&]() {  // accumulators drained: the MMA warp may start the next unit
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      };
      if constexpr (!STAGED) {
        // long reductions: the epilogue is a small share of a unit; per-row
        // direct stores (a thread writes its own row)
        u64 r0v[32], r1v[32];
        drain(0, r0v);
        if constexpr (NC > 1) drain(1, r1v);
        release();
        const i64 row = (i64)t.m0 + sp * 32 + lane;
        if (row < args.M) {
          u64* Crow = args.C + (i64)t.z * args.sC + row * args.ldc;
          const u64* Cin = args.Cin ? args.Cin + (i64)(t.z % args.zl) * args.sCin +
                                          (i64)(t.z / args.zl) * args.sCin_j + row * args.ldc
                                    : nullptr;
          const u64* src = atom ? (t.ks == 0 ? Cin : nullptr) : (Cin ? Cin : (args.accumulate ? Crow : nullptr));
#pragma unroll
          for (int q = 0; q < BN; ++q) {
            const int col = t.n0 + q;
            if (col < args.N) {
              const u64 v = (q < 32 ? r0v[q] : r1v[q - 32]) + (src ? src[col] : 0ull);
              if (atom)
                atomicAdd(reinterpret_cast<unsigned long long*>(Crow + col), (unsigned long long)v);
              else
                Crow[col] = v & args.msk;
            }
          }
        }
        continue;
      }
      // coalesced stores: each 32 x 32 block goes through this warp's smem
      // tile (row-owned -> column-owned), so a warp instruction writes 32
      // consecutive u64 of one output row. Chunk 0 is parked in shared memory
      // and chunk 1 in registers, so TMEM is released before any global
      // traffic.
      u64 hold[32];
      drain(c0, hold);
      if constexpr (NCW > 1) {
        u64 hold1[32];
        drain(1, hold1);
        release();  // TMEM free before waiting on any global traffic
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 32; ++q) stage[lane * 33 + q] += hold[q];  // thread = row, q = column
#pragma unroll
        for (int q = 0; q < 32; ++q) hold[q] = hold1[q];
      } else {
        release();
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 32; ++q) stage[lane * 33 + q] += hold[q];
      }
#pragma unroll
      for (int cc = 0; cc < NCW; ++cc) {
        const int c = c0 + cc;
        if (cc == 1) {  // chunk 1 waited in registers; its addend is read now
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 32; ++q) stage[lane * 33 + q] = hold[q];
        }
        __syncwarp();
        const int col = t.n0 + c * 32 + lane;
        const int rows = col < args.N ? rmax : 0;
        // all 32 addend loads in flight before the stores that use them
        u64 add[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) add[r] = (cc == 1 && src && r < rows) ? src[(i64)r * args.ldc + col] : 0ull;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          if (r < rows && !(args.dbg & 2)) {
            const u64 v = stage[r * 33 + lane] + add[r];
            u64* dst = Cz + (i64)r * args.ldc + col;
            if (atom)
              atomicAdd(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)v);
            else
              *dst = v & args.msk;
          }
        }
        __syncwarp();
      }
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

// 4 x 4 byte transpose of four u32 rows (out[j] byte r = a[r] byte j): 8 PRMT
__device__ __forceinline__ void bytes_transpose4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                                 uint32_t (&o)[4]) {
  const uint32_t t0 = __byte_perm(a0, a1, 0x5140), t1 = __byte_perm(a0, a1, 0x7362);
  const uint32_t t2 = __byte_perm(a2, a3, 0x5140), t3 = __byte_perm(a2, a3, 0x7362);
  o[0] = __byte_perm(t0, t2, 0x5410);
  o[1] = __byte_perm(t0, t2, 0x7632);
  o[2] = __byte_perm(t1, t3, 0x5410);
  o[3] = __byte_perm(t1, t3, 0x7632);
}

// 8 x 8 byte transpose: p[i] byte c = w[c] byte i (limb planes of 8 words),
// as four 4 x 4 transposes of the words' 32-bit halves (32 PRMT)
__device__ __forceinline__ void bytes_transpose8(const u64 (&w)[8], u64 (&p)[8]) {
  uint32_t a[4], b[4], c[4], d[4];
  bytes_transpose4((uint32_t)w[0], (uint32_t)w[1], (uint32_t)w[2], (uint32_t)w[3], a);
  bytes_transpose4((uint32_t)w[4], (uint32_t)w[5], (uint32_t)w[6], (uint32_t)w[7], b);
  bytes_transpose4((uint32_t)(w[0] >> 32), (uint32_t)(w[1] >> 32), (uint32_t)(w[2] >> 32), (uint32_t)(w[3] >> 32),
                   c);
  bytes_transpose4((uint32_t)(w[4] >> 32), (uint32_t)(w[5] >> 32), (uint32_t)(w[6] >> 32), (uint32_t)(w[7] >> 32),
                   d);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    p[i] = (u64)a[i] | ((u64)b[i] << 32);
    p[4 + i] = (u64)c[i] | ((u64)d[i] << 32);
  }
}

// non-transposed: each thread takes 8 consecutive columns of one row
__global__ void k_limb_split(uint8_t* __restrict__ out, const u64* __restrict__ A, i64 rows, i64 cols, i64 lda,
                             i64 plane, i64 Rpad, int tw) {
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
    uint8_t* dst = out + limb_off(r, c0, Rpad, tw);
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
                                                      i64 rows, i64 cols, i64 lda, i64 plane, i64 Rpad, int tw) {
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
    uint8_t* dst = out + limb_off(gn, gk, Rpad, tw);
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
  // planes are K-block tiled (limb_off): `pitch` = padded K bytes, plane =
  // Rpad * pitch; column offsets are not supported by the tiled layout
  CHECK_ARG(coff == 0 && pitch > 0 && plane % pitch == 0 && (pitch % 128 == 0 || pitch == 32 || pitch == 64));
  const i64 Rpad = plane / pitch;
  const int tw = limb_tw(pitch);
  if (rows == 0 || cols == 0) return MPX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (!trans) {
    k_limb_split<<<grid_for(rows * ((cols + 7) / 8)), MPX_THREADS, 0, s>>>(out, A, rows, cols, lda, plane, Rpad,
                                                                           tw);
  } else {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 63) / 64));
    CHECK_ARG(grid.y <= 65535);
    k_limb_split_t<<<grid, 256, 0, s>>>(out, A, rows, cols, lda, plane, Rpad, tw);
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
  const i64 total = (i64)L * Mpad * gpr;  // rows >= M written as zeros (tiled planes)
  GRID_STRIDE(t, total) {
    const i64 g = t % gpr;
    const i64 rl = t / gpr;
    const i64 r = rl % Mpad, l = rl / Mpad;
    const i64 c0 = g * 8;
    u64 w[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const i64 cc = c0 + c;
      w[c] = r >= M ? 0ull : (cc < Kd ? D[r * Kd + cc] : (cc < 2 * Kd ? A[l * a_ps + r * Kd + (cc - Kd)] : 0ull));
    }
    u64 pl[8];
    bytes_transpose8(w, pl);
    uint8_t* dst = A8 + (l * 8) * Mpad * Kpad + limb_off(r, c0, Mpad, limb_tw(Kpad));
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
    uint8_t* dst = B8 + ((i64)l * 8) * Npad * Kpad + limb_off(gn, gk, Npad, limb_tw(Kpad));
    const i64 plane = Npad * Kpad;
#pragma unroll
    for (int i = 0; i < 8; ++i) *reinterpret_cast<u64*>(dst + i * plane) = pl[i];
  }
}

extern "C" int mpx_beaver_limbs(uint8_t* A8, uint8_t* B8, const uint64_t* D, const uint64_t* E, const uint64_t* A,
                                int64_t a_ps, const uint64_t* B, int64_t b_ps, int L, int64_t M, int64_t K,
                                int64_t N, int64_t Mpad, int64_t Npad, int64_t Kpad, int p0, void* stream) {
  CHECK_ARG(A8 && B8 && D && E && A && B && L >= 1 && L <= 65535 && M >= 1 && K >= 1 && N >= 1);
  CHECK_ARG(Mpad >= M && Npad >= N && Kpad >= 2 * K && Kpad % 32 == 0);
  cudaStream_t s = (cudaStream_t)stream;
  const i64 ta = (i64)L * Mpad * ((Kpad + 7) / 8);
  // A side also zero-fills the K padding columns (groups beyond 2K read as 0)
  k_beaver_limbs_a<<<grid_for(ta), MPX_THREADS, 0, s>>>(A8, D, A, a_ps, L, M, K, Mpad, Kpad);
  dim3 grid((unsigned)((Npad + 31) / 32), (unsigned)((Kpad + 63) / 64), (unsigned)L);
  CHECK_ARG(grid.y <= 65535);
  k_beaver_limbs_b<<<grid, 256, 0, s>>>(B8, B, b_ps, E, p0, K, N, Npad, Kpad);
  return launch_status();
}

// --------------------------------------------------------------------------
// Fused Beaver mask + limb split for the all-parties-local (sim) session,
// where opening D = sum_l (X_l - T_l) (basic.py:66-70) is a local reduction:
//   S8[i][rho][kappa]    = limb i of S = (sum_l X_l - T_l) mod 2^w   (shared)
//   P8[l][i][rho][kappa] = limb i of T_l (+ S at party p0 when add_p0)
// X_l and T_l are logical R x K matrices at arbitrary (row, col) strides
// (transposed operands are read in place, each with its own coalesced
// mapping); output planes are K-major [Rpad][Kp], zero padded. This replaces
// mask kernel -> D in HBM -> limb kernel re-reading D once per party: S is
// written once as limbs and shared by every party's GEMM (split tensor maps
// in k_gemm_limbs_tc_pers).
struct MaskLimbArgs {
  const u64* X;
  i64 x_ps, x_sr, x_sc;
  const u64* T;
  i64 t_ps, t_sr, t_sc;
  uint8_t* S8;
  uint8_t* P8;
  i64 R, K, Rpad, Kp;
  u64 msk;
  int L, p0, add_p0, pad;
  i64 x_js, t_js;  // job strides (blockIdx.z = job) of X and T; planes follow per job
};

// A thread owns (row rr, 8-column group g) of a 32 (rows) x 64 (k) tile and
// gets its 8 consecutive-k values of a source either straight from global
// (k-fastest source: 64 contiguous bytes) or through a shared-memory
// transpose (any other strides: the tile is read along rows, coalesced).
template <bool KFAST>
__device__ __forceinline__ void ml_load8(u64 (&v)[8], const u64* __restrict__ src, i64 sr, i64 sc, i64 r0, i64 k0,
                                         i64 R, i64 K, u64 (*tile)[33], int t) {
  const int rr = t >> 3, g = t & 7;
  if constexpr (KFAST) {
    const i64 r = r0 + rr;
    const i64 kb = k0 + g * 8;
    const u64* p = src + r * sr + kb;
    if (r < R && kb + 8 <= K && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      // four 16-byte loads instead of eight 8-byte ones
#pragma unroll
      for (int c = 0; c < 8; c += 2) {
        const ulonglong2 q = __ldg(reinterpret_cast<const ulonglong2*>(p + c));
        v[c] = q.x;
        v[c + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const i64 k = kb + c;
        v[c] = (r < R && k < K) ? src[r * sr + k] : 0ull;
      }
    }
  } else {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int r2 = t & 31, k2 = (t >> 5) + 8 * p;
      const i64 r = r0 + r2, k = k0 + k2;
      tile[k2][r2] = (r < R && k < K) ? src[r * sr + k * sc] : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = tile[g * 8 + c][rr];
    __syncthreads();
  }
}

#ifndef MPX_ML_PREFETCH
#define MPX_ML_PREFETCH 1
#endif

// Pull this thread's part of a source tile towards L2 (ml_load8's addresses).
template <bool KFAST>
__device__ __forceinline__ void ml_prefetch(const u64* __restrict__ src, i64 sr, i64 sc, i64 r0, i64 k0, i64 R,
                                            i64 K, int t) {
  if constexpr (KFAST) {
    const i64 r = r0 + (t >> 3), k = k0 + (t & 7) * 8;
    if (r < R && k < K) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src + r * sr + k));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src + r * sr + min(k + 7, K - 1)));
    }
  } else {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const i64 r = r0 + (t & 31), k = k0 + (t >> 5) + 8 * p;
      if (r < R && k < K) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + r * sr + k * sc));
    }
  }
}

__device__ __forceinline__ void ml_emit(uint8_t* base, i64 plane, const u64 (&w)[8], i64 r0, i64 k0, i64 Kp,
                                        int t) {
  const int rr = t >> 3, g = t & 7;
  u64 pl[8];
  bytes_transpose8(w, pl);
  if (k0 + g * 8 >= Kp) return;  // Kp % 64 == 32: the last tile's upper half
  uint8_t* dst = base + limb_off(r0 + rr, k0 + g * 8, plane / Kp, limb_tw(Kp));
#pragma unroll
  for (int i = 0; i < 8; ++i) *reinterpret_cast<u64*>(dst + i * plane) = pl[i];
}

// Party limbs are emitted as soon as the party's material is loaded; party
// p0's, when S must be added, is emitted last from a second (L2-hot) read of
// its material tile, which keeps the register footprint small enough for
// three CTAs per SM.
template <bool XK, bool TK>
__device__ __forceinline__ void ml_tile(MaskLimbArgs a, i64 r0, i64 k0, i64 jb, u64 (*tile)[33]) {
  const int t = threadIdx.x;
  const i64 plane = a.Rpad * a.Kp;
  const bool defer = a.add_p0 && a.p0 >= 0;
  // job jb: its operands and its shared + per-party plane sets
  a.X += jb * a.x_js;
  a.T += jb * a.t_js;
  a.S8 += jb * 8 * plane;
  a.P8 += jb * (i64)a.L * 8 * plane;
  if (MPX_ML_PREFETCH)  // every party's source tiles in flight at once (the loop below is per-party serial)
    for (int l = 0; l < a.L; ++l) {
      ml_prefetch<XK>(a.X + (i64)l * a.x_ps, a.x_sr, a.x_sc, r0, k0, a.R, a.K, t);
      ml_prefetch<TK>(a.T + (i64)l * a.t_ps, a.t_sr, a.t_sc, r0, k0, a.R, a.K, t);
    }
  u64 s[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) s[c] = 0;
  for (int l = 0; l < a.L; ++l) {
    u64 v[8];
    ml_load8<XK>(v, a.X + (i64)l * a.x_ps, a.x_sr, a.x_sc, r0, k0, a.R, a.K, tile, t);
#pragma unroll
    for (int c = 0; c < 8; ++c) s[c] += v[c];
    ml_load8<TK>(v, a.T + (i64)l * a.t_ps, a.t_sr, a.t_sc, r0, k0, a.R, a.K, tile, t);
#pragma unroll
    for (int c = 0; c < 8; ++c) s[c] -= v[c];
    if (!(defer && l == a.p0)) ml_emit(a.P8 + (i64)l * 8 * plane, plane, v, r0, k0, a.Kp, t);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) s[c] &= a.msk;
  ml_emit(a.S8, plane, s, r0, k0, a.Kp, t);
  if (defer) {
    u64 v[8];
    ml_load8<TK>(v, a.T + (i64)a.p0 * a.t_ps, a.t_sr, a.t_sc, r0, k0, a.R, a.K, tile, t);
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = (v[c] + s[c]) & a.msk;
    ml_emit(a.P8 + (i64)a.p0 * 8 * plane, plane, v, r0, k0, a.Kp, t);
  }
}

// Row-major X and T (k contiguous) with L <= 3: every party's X_l and T_l
// words of the thread are loaded before any is used (2L x 64 bytes in flight
// per thread instead of 2 x 64: the party loop above is latency bound).
template <int LP>
__device__ __forceinline__ void ml_tile_pre(MaskLimbArgs a, i64 r0, i64 k0, i64 jb) {
  const int t = threadIdx.x;
  const i64 plane = a.Rpad * a.Kp;
  const bool defer = a.add_p0 && a.p0 >= 0;
  a.X += jb * a.x_js;
  a.T += jb * a.t_js;
  a.S8 += jb * 8 * plane;
  a.P8 += jb * (i64)a.L * 8 * plane;
  u64 xv[LP][8], tv[LP][8];
#pragma unroll
  for (int l = 0; l < LP; ++l) {
    ml_load8<true>(xv[l], a.X + (i64)l * a.x_ps, a.x_sr, 1, r0, k0, a.R, a.K, nullptr, t);
    ml_load8<true>(tv[l], a.T + (i64)l * a.t_ps, a.t_sr, 1, r0, k0, a.R, a.K, nullptr, t);
  }
  u64 s[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) s[c] = 0;
#pragma unroll
  for (int l = 0; l < LP; ++l) {
#pragma unroll
    for (int c = 0; c < 8; ++c) s[c] += xv[l][c] - tv[l][c];
    if (!(defer && l == a.p0)) ml_emit(a.P8 + (i64)l * 8 * plane, plane, tv[l], r0, k0, a.Kp, t);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) s[c] &= a.msk;
  ml_emit(a.S8, plane, s, r0, k0, a.Kp, t);
  if (defer) {
#pragma unroll
    for (int l = 0; l < LP; ++l)
      if (l == a.p0) {
        u64 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = (tv[l][c] + s[c]) & a.msk;
        ml_emit(a.P8 + (i64)l * 8 * plane, plane, v, r0, k0, a.Kp, t);
      }
  }
}

template <bool XK, bool TK>
__global__ void __launch_bounds__(256, 3) k_mask_limbs(MaskLimbArgs a) {
  __shared__ u64 tile[64][33];
  ml_tile<XK, TK>(a, (i64)blockIdx.x * 32, (i64)blockIdx.y * 64, blockIdx.z, tile);
}

// Both operand sides of a Beaver product in one launch: blocks [0, na) do
// side a's tiles, the rest side b's (each side's source layouts picked at run
// time; every block takes one branch, so its barriers stay uniform).
__device__ __forceinline__ void ml_tile_rt(const MaskLimbArgs& a, i64 r0, i64 k0, i64 jb, u64 (*tile)[33]) {
  const bool xk = a.x_sc == 1, tk = a.t_sc == 1;
  if (xk && tk)
    ml_tile<true, true>(a, r0, k0, jb, tile);
  else if (xk)
    ml_tile<true, false>(a, r0, k0, jb, tile);
  else if (tk)
    ml_tile<false, true>(a, r0, k0, jb, tile);
  else
    ml_tile<false, false>(a, r0, k0, jb, tile);
}

__device__ __forceinline__ void ml_tile_any(const MaskLimbArgs& a, i64 r0, i64 k0, i64 jb, u64 (*tile)[33]) {
  if (a.x_sc == 1 && a.t_sc == 1 && a.L <= 3) {
    switch (a.L) {
      case 1: ml_tile_pre<1>(a, r0, k0, jb); return;
      case 2: ml_tile_pre<2>(a, r0, k0, jb); return;
      default: ml_tile_pre<3>(a, r0, k0, jb); return;
    }
  }
  ml_tile_rt(a, r0, k0, jb, tile);
}

__global__ void __launch_bounds__(256, 2) k_mask_limbs2(const __grid_constant__ MaskLimbArgs a,
                                                        const __grid_constant__ MaskLimbArgs b, int ax, int na,
                                                        int bx) {
  __shared__ u64 tile[64][33];
  const int id = blockIdx.x;
  if (id < na)
    ml_tile_any(a, (i64)(id % ax) * 32, (i64)(id / ax) * 64, blockIdx.y, tile);
  else
    ml_tile_any(b, (i64)((id - na) % bx) * 32, (i64)((id - na) / bx) * 64, blockIdx.y, tile);
}

static void ml_pack(MaskLimbArgs& a, uint8_t* S8, uint8_t* P8, const uint64_t* X, int64_t x_ps, int64_t x_sr,
                    int64_t x_sc, const uint64_t* T, int64_t t_ps, int64_t t_sr, int64_t t_sc, int L, int64_t R,
                    int64_t K, int64_t Rpad, int64_t Kp, int p0, int add_p0, int width, int64_t x_js, int64_t t_js) {
  a.X = X;
  a.x_ps = x_ps;
  a.x_sr = x_sr;
  a.x_sc = x_sc;
  a.T = T;
  a.t_ps = t_ps;
  a.t_sr = t_sr;
  a.t_sc = t_sc;
  a.S8 = S8;
  a.P8 = P8;
  a.R = R;
  a.K = K;
  a.Rpad = Rpad;
  a.Kp = Kp;
  a.msk = ring_mask(width);
  a.L = L;
  a.p0 = p0;
  a.add_p0 = add_p0;
  a.pad = 0;
  a.x_js = x_js;
  a.t_js = t_js;
}

// Side A (X_l, A_l; logical m x k) and side B (Y_l^T, B_l^T; logical r x k,
// B_l + E at p0) of `jobs` products in ONE launch (sim mode).
extern "C" int mpx_mask_limbs2(uint8_t* SA8, uint8_t* PA8, const uint64_t* X, int64_t x_ps, int64_t x_sr,
                               int64_t x_sc, const uint64_t* A, int64_t a_ps, int64_t a_sr, int64_t a_sc,
                               int64_t M, int64_t Mpad, uint8_t* SB8, uint8_t* PB8, const uint64_t* Y, int64_t y_ps,
                               int64_t y_sr, int64_t y_sc, const uint64_t* B, int64_t b_ps, int64_t b_sr,
                               int64_t b_sc, int64_t N, int64_t Npad, int L, int64_t K, int64_t Kp, int p0,
                               int width, int jobs, int64_t x_js, int64_t a_js, int64_t y_js, int64_t b_js,
                               void* stream) {
  CHECK_ARG(SA8 && PA8 && X && A && SB8 && PB8 && Y && B && L >= 1 && M >= 1 && N >= 1 && K >= 1);
  CHECK_ARG(width >= 1 && width <= 64 && jobs >= 1 && jobs <= 65535);
  CHECK_ARG(Mpad >= M && Mpad % 32 == 0 && Npad >= N && Npad % 32 == 0 && Kp >= K && Kp % 32 == 0);
  MaskLimbArgs a, b;
  ml_pack(a, SA8, PA8, X, x_ps, x_sr, x_sc, A, a_ps, a_sr, a_sc, L, M, K, Mpad, Kp, p0, 0, width, x_js, a_js);
  ml_pack(b, SB8, PB8, Y, y_ps, y_sr, y_sc, B, b_ps, b_sr, b_sc, L, N, K, Npad, Kp, p0, 1, width, y_js, b_js);
  const i64 ky = (Kp + 63) / 64;
  const i64 ax = Mpad / 32, bx = Npad / 32;
  const i64 na = ax * ky, nb = bx * ky;
  CHECK_ARG(na + nb < (1ll << 31));
  k_mask_limbs2<<<dim3((unsigned)(na + nb), (unsigned)jobs), 256, 0, (cudaStream_t)stream>>>(a, b, (int)ax, (int)na,
                                                                                            (int)bx);
  return launch_status();
}

extern "C" int mpx_mask_limbs(uint8_t* S8, uint8_t* P8, const uint64_t* X, int64_t x_ps, int64_t x_sr, int64_t x_sc,
                              const uint64_t* T, int64_t t_ps, int64_t t_sr, int64_t t_sc, int L, int64_t R,
                              int64_t K, int64_t Rpad, int64_t Kp, int p0, int add_p0, int width, int jobs,
                              int64_t x_js, int64_t t_js, void* stream) {
  CHECK_ARG(S8 && P8 && X && T && L >= 1 && R >= 1 && K >= 1 && width >= 1 && width <= 64);
  CHECK_ARG(jobs >= 1 && jobs <= 65535);
  CHECK_ARG(Rpad >= R && Rpad % 32 == 0 && Kp >= K && Kp % 32 == 0);
  CHECK_ARG(Rpad / 32 <= 0x7FFFFFFF && (Kp + 63) / 64 <= 65535);
  MaskLimbArgs a;
  a.X = X;
  a.x_ps = x_ps;
  a.x_sr = x_sr;
  a.x_sc = x_sc;
  a.T = T;
  a.t_ps = t_ps;
  a.t_sr = t_sr;
  a.t_sc = t_sc;
  a.S8 = S8;
  a.P8 = P8;
  a.R = R;
  a.K = K;
  a.Rpad = Rpad;
  a.Kp = Kp;
  a.msk = ring_mask(width);
  a.L = L;
  a.p0 = p0;
  a.add_p0 = add_p0;
  a.pad = 0;
  a.x_js = x_js;
  a.t_js = t_js;
  dim3 grid((unsigned)(Rpad / 32), (unsigned)((Kp + 63) / 64), (unsigned)jobs);
  cudaStream_t s = (cudaStream_t)stream;
  const bool xk = x_sc == 1, tk = t_sc == 1;
  if (xk && tk)
    k_mask_limbs<true, true><<<grid, 256, 0, s>>>(a);
  else if (xk)
    k_mask_limbs<true, false><<<grid, 256, 0, s>>>(a);
  else if (tk)
    k_mask_limbs<false, true><<<grid, 256, 0, s>>>(a);
  else
    k_mask_limbs<false, false><<<grid, 256, 0, s>>>(a);
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

// `planes` K-block-tiled [Rpad][kbytes] limb planes (limb_off) as one 2D
// tensor of (planes * kbytes / tw * Rpad) rows of tw bytes.
// 3D map over K-block-tiled limb planes: (k within the tile, tile * Rpad +
// row, plane), box (bk, box_rows, box_planes) - consecutive limb planes of
// one k-block and row block in one TMA.
static int make_map3(CUtensorMap* map, const uint8_t* base, i64 planes, i64 Rpad, i64 kbytes, int box_rows, int bk,
                     int box_planes) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return MPX_ERR_CUDA;
  const int tw = limb_tw(kbytes);
  if (kbytes % tw != 0 || tw % bk != 0) return MPX_ERR_ARG;
  const i64 rows = (kbytes / tw) * Rpad;
  if (rows >= (1ll << 31) || planes >= (1ll << 31)) return MPX_ERR_ARG;
  cuuint64_t dims[3] = {(cuuint64_t)tw, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)tw, (cuuint64_t)(rows * tw)};
  cuuint32_t box[3] = {(cuuint32_t)bk, (cuuint32_t)box_rows, (cuuint32_t)box_planes};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = bk == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                          : (bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? MPX_OK : MPX_ERR_CUDA;
}

static int make_map(CUtensorMap* map, const uint8_t* base, i64 planes, i64 Rpad, i64 kbytes, int box_rows,
                    int bk = TC_BK) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return MPX_ERR_CUDA;
  const int tw = limb_tw(kbytes);
  if (kbytes % tw != 0 || tw % bk != 0) return MPX_ERR_ARG;
  const i64 rows = planes * (kbytes / tw) * Rpad;
  if (rows >= (1ll << 31)) return MPX_ERR_ARG;
  cuuint64_t dims[2] = {(cuuint64_t)tw, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)tw};
  cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = bk == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                          : (bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? MPX_OK : MPX_ERR_CUDA;
}

// C[z] (+)= sum_{i+j<=7} 2^(8(i+j)) A8[z][i] @ B8[z][j]^T  (mod 2^width)
// A8: [batch][8][Mpad][Kpad] u8, B8: [batch][8][Npad][Kpad] u8, zero padded;
// Mpad % 128 == 0, Npad % 64 == 0, Kpad % 128 == 0, Kpad <= 16384.
// Split-K for the persistent kernel: minimise waves x (k-blocks per unit +
// per-unit epilogue cost) over the slice counts that keep every slice within
// the exactness bound (<= 16384 of K per accumulator).
static int tcp_auto_split(i64 tiles, int nk_total, int sms, int bk = TC_BK) {
  const int need = (nk_total * bk + 16383) / 16384;
  int best = need;
  double best_cost = 1e30;
  for (int s = need; s <= nk_total && s <= 64; ++s) {
    const int per = (nk_total + s - 1) / s;
    const int se = (nk_total + per - 1) / per;
    if (se != s) continue;
    const i64 units = tiles * se;
    const i64 waves = (units + sms - 1) / sms;
    // epilogue (TMEM drain + stores) in k-blocks; atomics cost more than stores
    const double epi = (se > 1 ? 1.0 : 0.5) * (128.0 / bk);
    const double cost = (double)waves * (per + epi);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

// C[z] (+)= sum_{i+j<=7} 2^(8(i+j)) A8[z][i] @ B8[z][j]^T  (mod 2^width)
// A8: [batch][8][Mpad][Kpad] u8, B8: [batch][8][Npad][Kpad] u8, zero padded;
// Mpad % 128 == 0, Npad % 32 == 0, Kpad % 128 == 0. ksplit 0 = automatic
// (width 64 only), >= 1 = forced slice count.
template <int BK, int BN, bool ST, int EW = 4>
static int tcp_launch(unsigned g, cudaStream_t s, const CUtensorMap& mA, const CUtensorMap& mB,
                      const CUtensorMap& mA2, const CUtensorMap& mB2, const TcArgs& a, int batch) {
  static bool attr = false;
  constexpr int smem = tcp_smem_bytes(BK, BN, ST, EW);
  static_assert(smem <= 232448, "shared memory budget");
  if (!attr) {
    if (cudaFuncSetAttribute(k_gemm_limbs_tc_pers<BK, BN, ST, EW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess)
      return MPX_ERR_CUDA;
    attr = true;
  }
  k_gemm_limbs_tc_pers<BK, BN, ST, EW><<<g, 64 + 32 * EW, smem, s>>>(mA, mB, mA2, mB2, a, batch);
  return launch_status();
}

// C[z] (+)= sum_{i+j<=7} 2^(8(i+j)) A8[z][i] @ B8[z][j]^T  (mod 2^width)
// A8: [batch][8][Mpad][Kpad] u8, B8: [batch][8][Npad][Kpad] u8, zero padded;
// Mpad % 128 == 0, Npad % 32 == 0, Kpad % 32 == 0 (k-block = the largest of
// 128 / 64 / 32 bytes dividing Kpad). ksplit 0 = automatic (width 64 only),
// >= 1 = forced slice count.
static int gemm_limbs_impl(uint64_t* C, const uint8_t* A8, const uint8_t* B8, const uint8_t* A8s,
                           const uint8_t* B8s, int64_t batch, int64_t M, int64_t N, int64_t Mpad, int64_t Npad,
                           int64_t Kpad, int64_t ldc, int64_t sC, int accumulate, int width, int ksplit,
                           const uint64_t* Cin, int64_t sCin, void* stream, int zl = 0, int64_t sCin_j = 0) {
  if (zl <= 0) zl = (int)batch;  // one job: every z shares plane set 0
  CHECK_ARG(C && A8 && B8 && batch >= 1 && batch <= 65535 && M >= 1 && N >= 1 && width >= 1 && width <= 64);
  const bool split_ops = A8s != nullptr;
  CHECK_ARG(Mpad % TC_BM == 0 && Npad % 32 == 0 && Kpad % 32 == 0 && Kpad >= 32);
  const i64 kcols = split_ops ? Kpad / 2 : Kpad;  // split operands: each half its own plane set
  int bk = kcols % 128 == 0 ? 128 : (kcols % 64 == 0 ? 64 : 32);
  CHECK_ARG(!split_ops || (B8s && Kpad % 2 == 0 && kcols % 32 == 0));
  CHECK_ARG(M <= Mpad && N <= Npad && ldc >= N);
  CHECK_ARG(batch * 8 * Mpad < (1ll << 31) && batch * 8 * Npad < (1ll << 31));
  CHECK_ARG(!(Cin && accumulate));
  cudaStream_t s = (cudaStream_t)stream;
  const bool legacy = getenv("MPX_TC_LEGACY") != nullptr && !split_ops && bk == TC_BK;
  const int bn = Npad <= 32 ? 32 : 64;
  const i64 ptiles = (Mpad / TC_BM) * ((Npad + bn - 1) / bn) * batch;
  const int ks_req = ksplit;
  int nk_total = 0, nk_per = 0;
  auto plan = [&](int kb) -> int {
    nk_total = (int)(Kpad / kb);
    ksplit = ks_req;
    if (ksplit < 1) {
      if (width != 64) {
        ksplit = 1;
      } else if (legacy) {  // two waves of one-tile CTAs, every slice <= 16384 of K
        const i64 t64 = (Mpad / TC_BM) * (Npad / 64) * batch;
        const int need = (nk_total * TC_BK + 16383) / 16384;
        const int want = (int)max((i64)1, (2 * (i64)num_sms()) / max((i64)1, t64));
        ksplit = max(need, min(want, max(1, nk_total / 2)));
      } else {
        const char* force = getenv("MPX_TC_KSPLIT");  // sweeps / A-B timing
        ksplit = force ? max(1, atoi(force)) : tcp_auto_split(ptiles, nk_total, num_sms(), kb);
        ksplit = max(ksplit, (nk_total * kb + 16383) / 16384);
      }
    }
    if (ksplit > nk_total) ksplit = nk_total;
    nk_per = (nk_total + ksplit - 1) / ksplit;
    ksplit = (nk_total + nk_per - 1) / nk_per;
    return ksplit;
  };
  CHECK_ARG(ksplit >= 1 || width == 64 || Kpad <= 16384);
  plan(bk);
  const char* st = getenv("MPX_TC_STAGED");
  bool staged = st ? atoi(st) != 0 : (i64)nk_per * bk <= TCP_STAGED_MAX_KB * 128;
  if (!legacy && staged && bn == 64 && bk == 128) {
    bk = 64;  // staged 64-wide tiles run 64-byte k-blocks (room for 8 epilogue warps)
    plan(bk);
  }
  // exactness: each CTA's s32 diagonal accumulators see at most 16384 of K
  CHECK_ARG((i64)nk_per * bk <= 16384);
  // split-K adds partials with wrapping 64-bit atomics: exact mod 2^64 only
  CHECK_ARG(ksplit == 1 || width == 64);
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
  a.kb_half = split_ops ? (int)(kcols / bk) : 0;
  a.tw = limb_tw(kcols);
  a.nkt = (int)(kcols / a.tw);
  a.dbg = getenv("MPX_TC_DBG") ? atoi(getenv("MPX_TC_DBG")) : 0;
  a.zl = zl;
  a.sCin_j = sCin_j;
  CHECK_ARG(batch % zl == 0);
  CUtensorMap mapA, mapB, mapA2, mapB2;
  if (!legacy) {
    // split slices meet in C through atomics: start from zero unless C is
    // the accumulate operand (the addend rides on slice 0)
    if (ksplit > 1 && !accumulate) {
      if (ldc == N && sC == M * N) {  // one contiguous block: one memset node instead of `batch`
        if (cudaMemsetAsync(C, 0, (size_t)(batch * M * N * 8), s) != cudaSuccess) return MPX_ERR_CUDA;
      } else {
        for (i64 z = 0; z < batch; ++z)
          if (cudaMemset2DAsync(C + z * sC, (size_t)ldc * 8, 0, (size_t)N * 8, (size_t)M, s) != cudaSuccess)
            return MPX_ERR_CUDA;
      }
    }
    if (make_map3(&mapA, A8, batch * 8, Mpad, kcols, TC_BM, bk, MPX_TC_AP) != MPX_OK ||
        make_map3(&mapB, B8, batch * 8, Npad, kcols, bn, bk, 8) != MPX_OK)
      return MPX_ERR_CUDA;
    if (split_ops) {
      const i64 jobs = batch / zl;
      if (make_map3(&mapA2, A8s, jobs * 8, Mpad, kcols, TC_BM, bk, MPX_TC_AP) != MPX_OK ||
          make_map3(&mapB2, B8s, jobs * 8, Npad, kcols, bn, bk, 8) != MPX_OK)
        return MPX_ERR_CUDA;
    } else {
      mapA2 = mapA;
      mapB2 = mapB;
    }
    const i64 units = ptiles * ksplit;
    const unsigned g = (unsigned)min(units, (i64)num_sms());
    // coalesced (smem-staged) stores when the epilogue is a large share of a
    // unit; direct per-row stores for long reductions
    const int b = (int)batch;
    if (bk == 128 && bn == 64 && !staged)
      return tcp_launch<128, 64, false>(g, s, mapA, mapB, mapA2, mapB2, a, b);
    if (bk == 128 && bn == 32) return tcp_launch<128, 32, true>(g, s, mapA, mapB, mapA2, mapB2, a, b);
    if (bn == 64) {
      // staged 64-wide tiles: 64-byte k-blocks leave room for 8 epilogue
      // warps' transpose tiles (short reductions are epilogue-paced)
      if (bk == 32) return tcp_launch<32, 64, true, 8>(g, s, mapA, mapB, mapA2, mapB2, a, b);
      return tcp_launch<64, 64, true, 8>(g, s, mapA, mapB, mapA2, mapB2, a, b);
    }
    if (bk == 64) return tcp_launch<64, 32, true>(g, s, mapA, mapB, mapA2, mapB2, a, b);
    return tcp_launch<32, 32, true>(g, s, mapA, mapB, mapA2, mapB2, a, b);
  }
  // legacy one-tile-per-CTA kernels (MPX_TC_LEGACY=1, for A/B timing)
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(k_gemm_limbs_tc<TC_WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             tc_smem_bytes(TC_WIDE)) != cudaSuccess ||
        cudaFuncSetAttribute(k_gemm_limbs_tc<TC_NARROW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             tc_smem_bytes(TC_NARROW)) != cudaSuccess)
      return MPX_ERR_CUDA;
    attr_set = true;
  }
  if (make_map(&mapA, A8, batch * 8, Mpad, Kpad, TC_BM) != MPX_OK) return MPX_ERR_CUDA;
  if (ksplit > 1 && Cin) {
    for (i64 z = 0; z < batch; ++z)
      if (cudaMemcpy2DAsync(C + z * sC, (size_t)ldc * 8, Cin + z * sCin, (size_t)ldc * 8, (size_t)N * 8,
                            (size_t)M, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return MPX_ERR_CUDA;
    a.Cin = nullptr;
  } else if (ksplit > 1 && !accumulate) {
    for (i64 z = 0; z < batch; ++z)
      if (cudaMemset2DAsync(C + z * sC, (size_t)ldc * 8, 0, (size_t)N * 8, (size_t)M, s) != cudaSuccess)
        return MPX_ERR_CUDA;
  }
  const bool narrow = (Npad % 64 != 0) || nk_per <= 2;
  const int lbn = narrow ? 32 : 64;
  if (make_map(&mapB, B8, batch * 8, Npad, Kpad, lbn) != MPX_OK) return MPX_ERR_CUDA;
  dim3 grid((unsigned)((Npad / lbn) * (Mpad / TC_BM) * ksplit), 1, (unsigned)batch);
  if (narrow)
    k_gemm_limbs_tc<TC_NARROW><<<grid, 192, tc_smem_bytes(TC_NARROW), s>>>(mapA, mapB, a);
  else
    k_gemm_limbs_tc<TC_WIDE><<<grid, 192, tc_smem_bytes(TC_WIDE), s>>>(mapA, mapB, a);
  return launch_status();
}

extern "C" int mpx_gemm_limbs(uint64_t* C, const uint8_t* A8, const uint8_t* B8, int64_t batch, int64_t M,
                              int64_t N, int64_t Mpad, int64_t Npad, int64_t Kpad, int64_t ldc, int64_t sC,
                              int accumulate, int width, int ksplit, const uint64_t* Cin, int64_t sCin,
                              void* stream) {
  return gemm_limbs_impl(C, A8, B8, nullptr, nullptr, batch, M, N, Mpad, Npad, Kpad, ldc, sC, accumulate, width,
                         ksplit, Cin, sCin, stream);
}

// Beaver reconstruction from split limb operands (k_mask_limbs output):
// C[z] = Cin[z] + [S_A | P_A[z]] @ [P_B[z] ; S_B] with S_* shared by all z
// ([8][rows][Kh] planes) and P_* per party ([batch][8][rows][Kh]).
extern "C" int mpx_gemm_limbs_split(uint64_t* C, const uint8_t* PA8, const uint8_t* SA8, const uint8_t* PB8,
                                    const uint8_t* SB8, int64_t batch, int64_t M, int64_t N, int64_t Mpad,
                                    int64_t Npad, int64_t Kh, int64_t ldc, int64_t sC, int width, int ksplit,
                                    const uint64_t* Cin, int64_t sCin, int zl, int64_t sCin_j, void* stream) {
  CHECK_ARG(SA8 && SB8 && Kh % 32 == 0 && zl >= 1 && batch % zl == 0);
  return gemm_limbs_impl(C, PA8, PB8, SA8, SB8, batch, M, N, Mpad, Npad, 2 * Kh, ldc, sC, 0, width, ksplit, Cin,
                         sCin, stream, zl, sCin_j);
}

int mpx_gemm_tc(uint64_t*, const uint64_t*, const uint64_t*, int64_t, int64_t, int64_t, int64_t, int64_t,
                int64_t, int64_t, int, int, cudaStream_t) {
  return MPX_ERR_UNSUPPORTED;  // the u64 entry point needs caller scratch: see mpx_gemm_limbs
}

// --------------------------------------------------------------------------
// Thin sim-mode Beaver products on tcgen05 with the operand limbs built in
// shared memory (no limb planes in HBM):
//     Z_l = C_l + [D | A_l] @ [B_l + [l == p0] E ; E]        (basic.py:66-75)
// with D = sum_l X_l - A_l and E = sum_l Y_l - B_l (the openings are local
// sums: all parties live on this GPU), for K <= 32 and N <= 32 (LeNet's conv1
// forward: 73728 x 25 x 20 at three parties). One persistent CTA per SM:
//  * warps 0-3 (producers) own 32 rows each of a 128-row tile: lane k loads
//    column k of every party's X_l and A_l rows (all loads in flight at
//    once), accumulates D per column in registers and writes the u8 limb
//    tiles of A_l, then D, in the UMMA K-major 32-byte-swizzle layout (16-byte
//    chunk c of row r at chunk c ^ bit 2 of r) through a staging tile; lane 0
//    of warp 0 then issues per party the 72 limb MMAs of the two 32-byte
//    k-blocks (D x B'_l, then A_l x E; diagonal i+j accumulates in TMEM
//    columns 32(i+j) of the party's 256-column buffer, two buffers);
//  * warps 4-7 (epilogue) drain a party's 8 diagonals (tcgen05.ld), recombine
//    the limbs mod 2^64 onto the C_l addend and store Z_l, while the
//    producers already load the next tile.
// B'_l and E limb tiles (32 x 32 bytes each) are built once per CTA.
// Measured (tools/micro/thin_tc.py, conv1 forward): 94 us vs 110 us for the
// SIMT tall kernel; with loads, C/Z traffic and MMAs all disabled
// (MPX_THIN_DBG=7) the skeleton alone still takes 50 us: one CTA of eight
// warps per SM (the limb tiles take 160 KB) leaves the per-warp dependency
// chains exposed.
#define THIN_TA (128 * 32)  // one limb tile of the A side: 128 rows x 32 bytes
#define THIN_TB (32 * 32)   // one limb tile of the B side: 32 rows (N) x 32 bytes

struct ThinArgs {
  u64* Z;
  i64 sZ;
  const u64* C;
  i64 sC;
  const u64* X;
  i64 x_ps, x_sr, x_sc;
  const u64* A;
  i64 sA;
  const u64* Y;
  i64 y_ps, y_sr, y_sc;
  const u64* B;
  i64 sB;
  int M, K, N, p0, L;
  u64 msk;
  int dbg;  // timing experiments (MPX_THIN_DBG bits, wrong results): 1 no operand loads, 2 no C / Z traffic, 4 no MMA
};

__device__ __forceinline__ void thin_put16(uint8_t* tile, int r, int c, u64 lo, u64 hi) {
  const int pc = c ^ ((r >> 2) & 1);
  *reinterpret_cast<ulonglong2*>(tile + r * 32 + pc * 16) = make_ulonglong2(lo, hi);
}

// 16 values (k = 16c .. 16c+15) of one row -> 16-byte chunk c of row r of the
// 8 limb tiles at `base` (tile stride `ts` bytes)
__device__ __forceinline__ void thin_emit_chunk(uint8_t* base, int ts, int r, int c, const u64* v) {
  u64 p0[8], p1[8], w[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) w[q] = v[q];
  bytes_transpose8(w, p0);
#pragma unroll
  for (int q = 0; q < 8; ++q) w[q] = v[8 + q];
  bytes_transpose8(w, p1);
#pragma unroll
  for (int i = 0; i < 8; ++i) thin_put16(base + i * ts, r, c, p0[i], p1[i]);
}

#define TMEM_LD16(taddr, v)                                                                            \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
               "%14,%15}, [%16];"                                                                       \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),    \
                 "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), \
                 "=r"(v[14]), "=r"(v[15])                                                               \
               : "r"(taddr))

#define THIN_SP 33  // staging pitch (u64): odd, conflict-free row reads

constexpr int thin_smem_bytes(int L) {
  // D + L A_l tiles, L B'_l + E tiles, 4 producer warps' staging (32 x 33 u64), barriers
  return 8 * THIN_TA * (1 + L) + 8 * THIN_TB * (L + 1) + 4 * 32 * THIN_SP * 8 + 1024 + 1024;
}

// Roles (256 threads): warps 0-3 producers (warp w: rows 32w..32w+31 of the
// tile, all k; lane 0 of warp 0 also issues the tile's MMAs once the four
// have written it), warps 4-7 epilogue (TMEM lane quarter w - 4). Producers
// run one tile ahead of the epilogue: tile t+1's loads overlap tile t's
// drain and stores; its limb tiles are written once the MMAs of tile t have
// read theirs (sempty). Every tile's inputs are prefetched to L2 one tile
// ahead. (Eight warps: 255 registers per thread; a ninth warp would cap
// them at 168.)
template <int L>
__global__ void __launch_bounds__(256, 1) k_beaver_tc_thin(const __grid_constant__ ThinArgs a) {
  extern __shared__ __align__(1024) uint8_t thin_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)thin_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sD = smem;                          // 8 limb tiles
  uint8_t* sA = sD + 8 * THIN_TA;              // [L][8] limb tiles
  uint8_t* sBp = sA + L * 8 * THIN_TA;         // [L][8] B'_l limb tiles
  uint8_t* sE = sBp + L * 8 * THIN_TB;         // [8] E limb tiles
  u64* stg = reinterpret_cast<u64*>(sE + 8 * THIN_TB);                  // [4 warps][32][THIN_SP]
  uint64_t* tf = reinterpret_cast<uint64_t*>(stg + 4 * 32 * THIN_SP);  // [2] MMA done per TMEM buffer
  uint64_t* te = tf + 2;                                                // [2] buffer drained
  uint64_t* sempty = te + 2;  // [3] party l's MMAs done: its A_l limb tiles (and, for the last, D's) are free
  uint64_t* tready = sempty + 3;                                        // the producers wrote a tile's limb tiles
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tready + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K, N = a.N;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tf[b], 1);
      mbar_init(&te[b], 4);
    }
    for (int l = 0; l < 3; ++l) mbar_init(&sempty[l], 1);
    mbar_init(tready, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int tiles = (a.M + 127) / 128;
  // L2 prefetch of a tile's X_l / A_l rows (warps 0-3: their own 32 rows)
  auto prefetch_tile = [&](int t) {
    const i64 wr0 = (i64)t * 128 + warp * 32;
    const int rows = (int)max((i64)0, min((i64)32, (i64)a.M - wr0));
    for (int l = 0; l < L; ++l) {
      const u64* Xl = a.X + l * a.x_ps + wr0 * a.x_sr;
      const u64* Al = a.A + l * a.sA + wr0 * (i64)K;
      for (int r = lane; r < rows; r += 32) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(Al + (i64)r * K));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(Al + (i64)r * K + K - 1));
        if (a.x_sc == 1) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(Xl + (i64)r * a.x_sr));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(Xl + (i64)r * a.x_sr + K - 1));
        }
      }
    }
  };
  if (warp < 4 && blockIdx.x < tiles) prefetch_tile(blockIdx.x);
  // B side once per CTA: E = sum_l Y_l - B_l; B'_l = B_l + [l == p0] E (rows = n,
  // bytes = k). E and every B_l are first gathered into the (still free) staging area.
  if (warp < 4) {
    u64* Es = stg;            // [32 k][32 n]
    u64* Bs = stg + 32 * 32;  // [L][32 k][32 n]
    for (int idx = threadIdx.x; idx < 32 * 32; idx += 128) {
      const int k = idx >> 5, n = idx & 31;
      const bool ok = k < K && n < N;
      u64 bv[L], yv[L];
#pragma unroll
      for (int l = 0; l < L; ++l) {
        bv[l] = ok ? __ldg(a.B + l * a.sB + (i64)k * N + n) : 0ull;
        yv[l] = ok ? __ldg(a.Y + l * a.y_ps + (i64)k * a.y_sr + (i64)n * a.y_sc) : 0ull;
      }
      u64 e = 0;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        e += yv[l] - bv[l];
        Bs[l * 1024 + idx] = bv[l];
      }
      Es[idx] = e;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    for (int job = threadIdx.x; job < (L + 1) * 64; job += 128) {
      const int n = job & 31, c = (job >> 5) & 1, which = job >> 6;  // which < L: B'_which, == L: E
      u64 v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = 16 * c + q;
        const u64 e = Es[k * 32 + n];
        v[q] = which == L ? e : Bs[which * 1024 + k * 32 + n] + (which == a.p0 ? e : 0ull);
      }
      thin_emit_chunk(which == L ? sE : sBp + which * 8 * THIN_TB, THIN_TB, n, c, v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, 128;" ::: "memory");  // staging free again
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;
  const uint32_t idesc_base = (2u << 4) | ((uint32_t)(128 >> 4) << 24);

  if (warp < 4) {
    // ---------------- producers ----------------
    u64* sx = stg + warp * 32 * THIN_SP;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      if (t + (int)gridDim.x < tiles) prefetch_tile(t + gridDim.x);
      const i64 wr0 = (i64)t * 128 + warp * 32;
      const int rows = (int)max((i64)0, min((i64)32, (i64)a.M - wr0));
      // lane = column k: D is accumulated per column in registers (dcol[r] =
      // D[row r][k]); each party's A_l tile and finally D go to row-owned
      // lanes through the staging tile for the limb emission.
      const bool kok = lane < K;
      u64 dcol[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) dcol[r] = 0;
      for (int l = 0; l < L; ++l) {
        const u64* __restrict__ Xl = a.X + l * a.x_ps + wr0 * a.x_sr + (i64)lane * a.x_sc;
        const u64* __restrict__ Al = a.A + l * a.sA + wr0 * (i64)K + lane;
        u64 t[32], tx[32];  // X_l's and A_l's loads all in flight together
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const bool ld = kok && r < rows && !(a.dbg & 1);
          tx[r] = ld ? __ldg(Xl + (i64)r * a.x_sr) : 0ull;
          t[r] = ld ? __ldg(Al + (i64)r * K) : 0ull;
        }
#pragma unroll
        for (int r = 0; r < 32; ++r) dcol[r] += tx[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          dcol[r] -= t[r];
          sx[r * THIN_SP + lane] = t[r];
        }
        __syncwarp();
        // the previous tile's MMAs must have read the limb tiles
        if (it > 0) mbar_wait(&sempty[l], (uint32_t)((it - 1) & 1));  // the previous tile's party-l MMAs read theirs
#pragma unroll
        for (int c = 0; c < 2; ++c) {  // A_l row (lane = row): 16 words at a time
          u64 v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = sx[lane * THIN_SP + 16 * c + q];
          thin_emit_chunk(sA + l * 8 * THIN_TA, THIN_TA, warp * 32 + lane, c, v);
        }
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 32; ++r) sx[r * THIN_SP + lane] = dcol[r] & a.msk;
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        u64 v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = sx[lane * THIN_SP + 16 * c + q];
        thin_emit_chunk(sD, THIN_TA, warp * 32 + lane, c, v);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tready);  // the MMAs are issued by the epilogue side (warp 4)
    }
  } else {
    // ---------------- epilogue: drain, recombine, Z_l = C_l + acc (a thread = a row) ----------------
    const int rq = warp - 4;
    int job = 0, it = 0;
    // ---- MMA issue (warp 4, lane 0): per party two k-blocks of 36 limb products.
    // A_i x [B_0 .. B_{7-i}] is ONE MMA of N = 32 (8 - i): the B limb tiles are
    // consecutive rows of one operand and diagonals i..7 adjacent TMEM column
    // blocks. Issuing from the epilogue side keeps the producers loading the
    // next tile while a TMEM buffer waits to be drained.
    auto issue = [&](int jb, int l) {
      const int buf = jb & 1;
      if (jb >= 2) mbar_wait(&te[buf], (uint32_t)(((jb - 2) >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dt = tmem_base + (uint32_t)(buf * 256);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t id = idesc_base | ((uint32_t)((32 * (8 - i)) >> 3) << 17);
        if (!(a.dbg & 4)) {
          mma_i8(dt + (uint32_t)(i * 32), umma_desc_sw<32>(smem_u32(sD + i * THIN_TA)),
                 umma_desc_sw<32>(smem_u32(sBp + l * 8 * THIN_TB)), id, i > 0 ? 1u : 0u);
          mma_i8(dt + (uint32_t)(i * 32), umma_desc_sw<32>(smem_u32(sA + (l * 8 + i) * THIN_TA)),
                 umma_desc_sw<32>(smem_u32(sE)), id, 1u);
        }
      }
      umma_commit(&tf[buf]);
      umma_commit(&sempty[l]);  // party l's A_l tiles (after the last party: D's too) may be overwritten
    };
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const i64 row = (i64)t * 128 + rq * 32 + lane;
      if (rq == 0 && lane == 0) {  // the tile's first party, once the producers wrote it
        mbar_wait(tready, (uint32_t)(it & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        issue(job, 0);
      }
      __syncwarp();
      for (int l = 0; l < L; ++l, ++job) {
        const int buf = job & 1;
        const u64* __restrict__ Cl = a.C + l * a.sC + row * (i64)N;
        u64* __restrict__ Zl = a.Z + l * a.sZ + row * (i64)N;
        u64 acc[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = (q < N && row < a.M && !(a.dbg & 2)) ? __ldg(Cl + q) : 0ull;  // addend first
        mbar_wait(&tf[buf], (uint32_t)((job >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (rq == 0 && lane == 0 && l + 1 < L) issue(job + 1, l + 1);  // next party's MMAs under this drain
        __syncwarp();
        // two diagonals' TMEM loads in flight per wait (four waits per party)
#pragma unroll
        for (int d0 = 0; d0 < 8; d0 += 2) {
          uint32_t v0[32], v1[32];
          const uint32_t ta = tmem_base + ((uint32_t)(rq * 32) << 16) + (uint32_t)(buf * 256 + d0 * 32);
          TMEM_LD32(ta, v0);
          TMEM_LD32(ta + 32, v1);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 32; ++q) acc[q] += ((u64)v0[q] << (8 * d0)) + ((u64)v1[q] << (8 * d0 + 8));
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&te[buf]);
        if (row < a.M && !(a.dbg & 2)) {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (q < N) Zl[q] = acc[q] & a.msk;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

template <int L>
static int thin_launch(const ThinArgs& a, cudaStream_t s) {
  static bool attr = false;
  constexpr int smem = thin_smem_bytes(L);
  static_assert(smem <= 232448, "shared memory budget");
  if (!attr) {
    if (cudaFuncSetAttribute(k_beaver_tc_thin<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return MPX_ERR_CUDA;
    attr = true;
  }
  const int tiles = (a.M + 127) / 128;
  k_beaver_tc_thin<L><<<min(tiles, num_sms()), 256, smem, s>>>(a);
  return launch_status();
}

// Z [L][M][N], C [L][M][N], A [L][M][K], B [L][K][N] (party strides sZ, sC,
// sA, sB); X, Y logical M x K and K x N share views at (party, row, col)
// strides. K <= 32, N <= 32, 2 <= L <= 3 (all parties local), width 64.
extern "C" int mpx_beaver_tc_thin(uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* X,
                                  int64_t x_ps, int64_t x_sr, int64_t x_sc, const uint64_t* A, int64_t sA,
                                  const uint64_t* Y, int64_t y_ps, int64_t y_sr, int64_t y_sc, const uint64_t* B,
                                  int64_t sB, int L, int64_t M, int64_t K, int64_t N, int p0, int width,
                                  void* stream) {
  CHECK_ARG(Z && C && X && A && Y && B && M >= 1 && K >= 1 && K <= 32 && N >= 1 && N <= 32);
  CHECK_ARG(L >= 2 && L <= 3 && p0 >= -1 && p0 < L && width >= 1 && width <= 64 && M < (1ll << 31));
  ThinArgs a;
  a.Z = Z;
  a.sZ = sZ;
  a.C = C;
  a.sC = sC;
  a.X = X;
  a.x_ps = x_ps;
  a.x_sr = x_sr;
  a.x_sc = x_sc;
  a.A = A;
  a.sA = sA;
  a.Y = Y;
  a.y_ps = y_ps;
  a.y_sr = y_sr;
  a.y_sc = y_sc;
  a.B = B;
  a.sB = sB;
  a.M = (int)M;
  a.K = (int)K;
  a.N = (int)N;
  a.p0 = p0;
  a.L = L;
  a.msk = ring_mask(width);
  a.dbg = getenv("MPX_THIN_DBG") ? atoi(getenv("MPX_THIN_DBG")) : 0;
  cudaStream_t s = (cudaStream_t)stream;
  return L == 2 ? thin_launch<2>(a, s) : thin_launch<3>(a, s);
}

// --------------------------------------------------------------------------
// Long-K small sim-mode Beaver products on tcgen05 (weight gradients of thin
// layers: LeNet conv1 dW = cols^T @ dZ, 25 x 73728 x 20 at three parties):
//     Z_l = C_l + D @ B_l + A_l @ E + [l == p0] D @ E        (basic.py:66-75)
// for M, N <= 32 and any K. The K range is split over one CTA per SM. Each
// CTA streams its k-blocks (32 k) of every party's X_l, A_l (M side) and
// Y_l, B_l (N side) into shared memory -- TMA bulk copies (one per party for
// a contiguous run, one per 256-byte row otherwise), two raw buffers so block
// t + 2 lands while block t is converted -- forms D and E, and writes the u8
// limb tiles of two 128-row MMA families that stack the parties along M:
//   F1: [A_0; A_1; A_2; D]          x E      -> A_l @ E and D @ E
//   F2: [B_0^T; B_1^T; B_2^T; -]    x D^T    -> (D @ B_l)^T
// (32 rows per group; limb i of the stack times B limbs 0 .. 7-i as one MMA of
// N = 32 (8 - i), diagonal i + j accumulating in TMEM columns 32 (i + j):
// F1 in columns 0-255, F2 in 256-511). The accumulators stay in TMEM over the
// CTA's whole K range (at most 512 blocks per CTA keeps every diagonal exact
// in the bits it contributes mod 2^64); the epilogue recombines the limbs,
// transposes F2 through shared memory and writes the CTA's partial product;
// a second kernel sums the partials onto C_l. Width 64 only. Unused stack rows
// / columns carry garbage that only reaches ignored accumulator entries.
#define LONG_KMAJ 0   // the block is one contiguous run: (row, k) at (kb0 + k) R + row -> [k][R]
#define LONG_ROW16 1  // k is the unit stride, rows 16-byte aligned -> [row][LONG_RP]
#define LONG_ROW8 2   // anything else (8-byte copies) -> [row][LONG_RP]
#define LONG_ROWT 3   // k is the unit stride, one 3D tensor-map TMA box per 16-k half -> [half][party][row][16], 128B swizzle
#define LONG_RP 34    // row pitch (words): 16-byte rows, conflict-free 16-byte reads down a column

struct LongArgs {
  u64* W;  // partial products [grid][L][M][N]
  const u64* X;
  i64 x_ps, x_sr, x_sc;
  const u64* A;
  i64 sA;
  const u64* Y;
  i64 y_ps, y_sr, y_sc;
  const u64* B;
  i64 sB;
  int M, K, N, p0, L;
  int nkb;       // k-blocks in total (CTA b takes blocks b, b + grid, ...)
  int mode[4];   // layout / fill per family X, A, Y, B
  int off[4];    // word offset of each family in a raw buffer
  int rw;        // words per raw buffer
  int txb;       // bytes the bulk copies of one full block deliver
  int tma;       // full blocks arrive by bulk / tensor copies (no ROW8 family)
  int hb;        // LONG_ROWT: words per half box (1024-byte padded)
  int dbg;       // timing experiments (MPX_LONG_DBG bits, wrong results): 1 no operand loads, 2 no conversion, 4 no MMA
};

#define LONG_TA 4096  // one 128-row limb tile (32 bytes of k per row)
#define LONG_TB 1024  // one 32-row limb tile
#define LONG_LIMB_BYTES (2 * 8 * LONG_TA + 2 * 8 * LONG_TB)

static int long_hb_words(int L, int R) { return (L * R * 128 + 1023) / 1024 * 128; }
static int long_fam_words(int mode, int L, int R) {
  return mode == LONG_ROWT ? 2 * long_hb_words(L, R) : L * R * (mode == LONG_KMAJ ? 32 : LONG_RP);
}
static int long_smem_bytes(int rw) { return 1024 + LONG_LIMB_BYTES + 2 * rw * 8 + 64; }

// word of element (party l, row, k) within a family's region
__device__ __forceinline__ int long_idx(int mode, int R, int hb, int l, int row, int k) {
  const int g = l * R + row;
  if (mode == LONG_KMAJ) return l * R * 32 + k * R + row;
  if (mode == LONG_ROWT) return (k >> 4) * hb + g * 16 + ((((k & 15) >> 1) ^ (g & 7)) << 1) + (k & 1);
  return g * LONG_RP + k;
}

__device__ __forceinline__ void cp_async8z(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(ok ? 8u : 0u) : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Bulk-copy fill of one family for a full k-block, by warp 0's lanes (the
// expect_tx was posted before).
template <int L>
__device__ __forceinline__ void long_bulk(int mode, uint32_t dst, const u64* __restrict__ g, i64 ps, i64 sr, int R,
                                          int kb0, uint64_t* bar, int lane) {
  if (mode == LONG_KMAJ) {
    if (lane < L) bulk_g2s(dst + 8u * (uint32_t)(lane * R * 32), g + lane * ps + (i64)kb0 * R, (uint32_t)(R * 256), bar);
  } else {
    for (int q = lane; q < L * R; q += 32) {
      const int l = q / R, row = q - l * R;
      bulk_g2s(dst + 8u * (uint32_t)(q * LONG_RP), g + l * ps + row * sr + kb0, 256u, bar);
    }
  }
}

// cp.async fill of one family (partial last block, or ROW8 families), all
// threads; words past K are zero-filled. Element (row, k) of party l is at
// g + l ps + row sr + k sk.
template <int L>
__device__ __forceinline__ void long_fill(int mode, uint32_t dst, const u64* __restrict__ g, i64 ps, i64 sr, i64 sk,
                                          int R, int kb0, int K, int hb) {
#pragma unroll
  for (int l = 0; l < L; ++l)
    for (int q = threadIdx.x; q < 32 * R; q += 256) {
      int row, k;
      if (mode == LONG_KMAJ) k = q / R, row = q - k * R;
      else row = q >> 5, k = q & 31;
      const int gk = kb0 + k;
      const bool ok = gk < K;
      cp_async8z(dst + 8u * (uint32_t)long_idx(mode, R, hb, l, row, k),
                 ok ? g + l * ps + row * sr + (i64)gk * sk : g, ok);
    }
}

template <int L>
__global__ void __launch_bounds__(256, 1) k_beaver_tc_long(const __grid_constant__ LongArgs a,
                                                         const __grid_constant__ CUtensorMap mapA) {
  extern __shared__ __align__(1024) uint8_t long_raw_sm[];
  // 1024-aligned, derived from the shared array (keeps ld / st.shared)
  uint8_t* smem = long_raw_sm + ((1024u - (smem_u32(long_raw_sm) & 1023u)) & 1023u);
  uint8_t* f1a = smem;                 // [8] 128-row limb tiles: A_0 | A_1 | A_2 | D
  uint8_t* f2a = f1a + 8 * LONG_TA;    // [8] 128-row limb tiles: B_0^T | B_1^T | B_2^T | -
  uint8_t* f1b = f2a + 8 * LONG_TA;    // [8] 32-row limb tiles: E^T (rows n)
  uint8_t* f2b = f1b + 8 * LONG_TB;    // [8] 32-row limb tiles: D (rows m)
  u64* raw0 = reinterpret_cast<u64*>(f2b + 8 * LONG_TB);
  const int m = a.M, n = a.N, RW = a.rw;
  uint64_t* sdone = reinterpret_cast<uint64_t*>(raw0 + 2 * RW);
  uint64_t* full = sdone + 1;  // [2] bulk copies of raw buffer b landed
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(full + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // k-blocks blockIdx.x, + gridDim.x, ...: at any moment the CTAs stream
  // neighbouring blocks (spread over the DRAM channels, no camping on one stride)
  const int G = gridDim.x;
  const int nb = blockIdx.x < a.nkb ? (a.nkb - 1 - blockIdx.x) / G + 1 : 0;
  const int mx = a.mode[0], ma = a.mode[1], my = a.mode[2], mb = a.mode[3];

  if (threadIdx.x == 0) {
    mbar_init(sdone, 1);
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  } else if (warp == 1 && lane == 0 && ma == LONG_ROWT) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;
  auto is_bulk = [&](int t) { return a.tma && ((int)blockIdx.x + t * G + 1) * 32 <= a.K; };
  auto issue = [&](int t) {
    if (a.dbg & 1) return;
    const uint32_t base = smem_u32(raw0 + (t & 1) * RW);
    const int kb0 = ((int)blockIdx.x + t * G) * 32;
    if (is_bulk(t)) {
      if (warp == 0) {
        uint64_t* bar = &full[t & 1];
        if (lane == 0) mbar_expect_tx(bar, (uint32_t)a.txb);
        __syncwarp();
        long_bulk<L>(mx, base + 8u * a.off[0], a.X, a.x_ps, a.x_sr, m, kb0, bar, lane);
        if (ma == LONG_ROWT) {
          if (lane == 0) {
            u64* fa = raw0 + (t & 1) * RW + a.off[1];
            tma_load_3d(fa, &mapA, bar, kb0, 0, 0);
            tma_load_3d(fa + a.hb, &mapA, bar, kb0 + 16, 0, 0);
          }
        } else {
          long_bulk<L>(ma, base + 8u * a.off[1], a.A, a.sA, a.K, m, kb0, bar, lane);
        }
        long_bulk<L>(my, base + 8u * a.off[2], a.Y, a.y_ps, a.y_sc, n, kb0, bar, lane);
        long_bulk<L>(mb, base + 8u * a.off[3], a.B, a.sB, 1, n, kb0, bar, lane);
      }
    } else {
      long_fill<L>(mx, base + 8u * a.off[0], a.X, a.x_ps, a.x_sr, a.x_sc, m, kb0, a.K, a.hb);
      long_fill<L>(ma, base + 8u * a.off[1], a.A, a.sA, a.K, 1, m, kb0, a.K, a.hb);
      long_fill<L>(my, base + 8u * a.off[2], a.Y, a.y_ps, a.y_sc, a.y_sr, n, kb0, a.K, a.hb);
      long_fill<L>(mb, base + 8u * a.off[3], a.B, a.sB, 1, a.N, n, kb0, a.K, a.hb);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  // the first two blocks' copies; the other warps go straight to block 0's
  // full barrier (cp.async blocks are waited for by every thread below)
  if (nb > 0) issue(0);
  if (nb > 1) issue(1);
  const uint32_t idesc_base = (2u << 4) | ((uint32_t)(128 >> 4) << 24);
  // conversion units: (row of an operand family, 16-k chunk); rows enumerate
  // A_l (L m), D (m, in party 0's X slot), E^T (n, in party 0's Y slot), B_l^T (L n)
  const int urows = L * m + m + n + L * n;
  for (int t = 0; t < nb; ++t) {
    if (is_bulk(t)) {
      if (!(a.dbg & 1)) mbar_wait(&full[t & 1], (uint32_t)((t >> 1) & 1));
    } else {
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    u64* rb = raw0 + (t & 1) * RW;
    u64* rX = rb + a.off[0];
    const u64* rA = rb + a.off[1];
    u64* rY = rb + a.off[2];
    const u64* rB = rb + a.off[3];
    // openings, element-wise: D = sum_l X_l - A_l over X_0, E = sum_l Y_l - B_l
    // over Y_0 (in X's / Y's layout). Warp w: k = w, w + 8, w + 16, w + 24; lane = row.
    if (!(a.dbg & 2)) {
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int R = f ? n : m, fx = f ? my : mx, fa = f ? mb : ma;
        u64* xs = f ? rY : rX;
        const u64* as = f ? rB : rA;
        if (lane < R) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = warp + 8 * j;
            u64 d = 0;
#pragma unroll
            for (int l = 0; l < L; ++l)
              d += xs[long_idx(fx, R, a.hb, l, lane, k)] - as[long_idx(fa, R, a.hb, l, lane, k)];
            xs[long_idx(fx, R, a.hb, 0, lane, k)] = d;
          }
        }
      }
    }
    __syncthreads();
    if (t > 0) mbar_wait(sdone, (uint32_t)((t - 1) & 1));  // the previous block's MMAs read their tiles
    for (int u = threadIdx.x; u < ((a.dbg & 2) ? 0 : 2 * urows); u += 256) {
      const int c = u >= urows ? 1 : 0, row = u - c * urows;
      const u64* src;
      uint8_t* dst;
      int ts, r, tr, md, R, l = 0;
      if (row < L * m) {  // A_l row -> F1 group l
        l = row / m;
        r = row - l * m;
        src = rA, dst = f1a, ts = LONG_TA, tr = 32 * l + r, md = ma, R = m;
      } else if (row < L * m + m) {  // D row -> F1 group 3 (and F2's B operand below)
        r = row - L * m;
        src = rX, dst = f1a, ts = LONG_TA, tr = 96 + r, md = mx, R = m;
      } else if (row < L * m + m + n) {  // E^T row -> F1's B operand
        r = row - L * m - m;
        src = rY, dst = f1b, ts = LONG_TB, tr = r, md = my, R = n;
      } else {  // B_l^T row -> F2 group l
        const int rr = row - L * m - m - n;
        l = rr / n;
        r = rr - l * n;
        src = rB, dst = f2a, ts = LONG_TA, tr = 32 * l + r, md = mb, R = n;
      }
      u64 v[16];
      if (md == LONG_KMAJ) {
        const u64* sp = src + l * R * 32 + r;
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = sp[(16 * c + q) * R];
      } else if (md == LONG_ROWT) {
        const int g = l * R + r;
        const ulonglong2* sr = reinterpret_cast<const ulonglong2*>(src + c * a.hb + g * 16);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const ulonglong2 p = sr[q ^ (g & 7)];
          v[2 * q] = p.x;
          v[2 * q + 1] = p.y;
        }
      } else {
        const ulonglong2* sr = reinterpret_cast<const ulonglong2*>(src + (l * R + r) * LONG_RP + 16 * c);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const ulonglong2 p = sr[q];
          v[2 * q] = p.x;
          v[2 * q + 1] = p.y;
        }
      }
      thin_emit_chunk(dst, ts, tr, c, v);
      if (row >= L * m && row < L * m + m) thin_emit_chunk(f2b, LONG_TB, r, c, v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // tiles written; raw buffer t & 1 consumed
    if (t + 2 < nb) issue(t + 2);
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int i = 0; i < ((a.dbg & 4) ? 0 : 8); ++i) {
        const uint32_t id = idesc_base | ((uint32_t)((32 * (8 - i)) >> 3) << 17);
        const uint32_t acc = (t > 0 || i > 0) ? 1u : 0u;
        mma_i8(tmem_base + (uint32_t)(i * 32), umma_desc_sw<32>(smem_u32(f1a + i * LONG_TA)),
               umma_desc_sw<32>(smem_u32(f1b)), id, acc);
        mma_i8(tmem_base + (uint32_t)(256 + i * 32), umma_desc_sw<32>(smem_u32(f2a + i * LONG_TA)),
               umma_desc_sw<32>(smem_u32(f2b)), id, acc);
      }
      umma_commit(sdone);
    }
  }
  if (nb > 0) {
    mbar_wait(sdone, (uint32_t)((nb - 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // F2 (rows n) and D @ E (rows 96..) through shared memory (the limb
    // tiles: every MMA has completed)
    u64* S2 = reinterpret_cast<u64*>(smem);   // [L][32 m][33]
    u64* SDE = S2 + L * 32 * 33;              // [32 m][33]
    auto drain = [&](uint32_t col0, u64 (&val)[32]) {
#pragma unroll
      for (int q = 0; q < 32; ++q) val[q] = 0;
      const uint32_t ta = tmem_base + ((uint32_t)(warp * 32) << 16) + col0;
#pragma unroll
      for (int d0 = 0; d0 < 8; d0 += 2) {
        uint32_t v0[32], v1[32];
        TMEM_LD32(ta + (uint32_t)(d0 * 32), v0);
        TMEM_LD32(ta + (uint32_t)(d0 * 32 + 32), v1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 32; ++q) val[q] += ((u64)v0[q] << (8 * d0)) + ((u64)v1[q] << (8 * d0 + 8));
      }
    };
    if (warp < L) {  // lane = column n of (D B_l)^T
      u64 val[32];
      drain(256, val);
      if (lane < n) {
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < m) S2[(warp * 32 + q) * 33 + lane] = val[q];
      }
    } else if (warp == 3 && a.p0 >= 0) {  // lane = row m of D @ E
      u64 val[32];
      drain(0, val);
#pragma unroll
      for (int q = 0; q < 32; ++q) SDE[lane * 33 + q] = val[q];
    }
    __syncthreads();
    if (warp < L) {  // lane = row m of A_l @ E -> this CTA's partial of Z_l
      u64 val[32];
      drain(0, val);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        u64 v = val[q] + S2[(warp * 32 + lane) * 33 + q];
        if (warp == a.p0) v += SDE[lane * 33 + q];
        S2[(warp * 32 + lane) * 33 + q] = v;
      }
      __syncwarp();
      u64* wp = a.W + ((i64)blockIdx.x * L + warp) * m * n;  // row-major m x n, coalesced
      for (int e = lane; e < m * n; e += 32) {
        const int r = e / n, cc = e - r * n;
        wp[e] = S2[(warp * 32 + r) * 33 + cc];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// Z_l = C_l + sum over the CTAs' partials: a CTA takes 32 output words, its
// eight warps every eighth partial (all loads of a warp in flight together),
// then a shared-memory sum across the warps
__global__ void __launch_bounds__(256) k_long_reduce(u64* __restrict__ Z, i64 sZ, const u64* __restrict__ C, i64 sC,
                                                     const u64* __restrict__ W, int L, int mn, int parts) {
  __shared__ u64 red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int o = blockIdx.x * 32 + lane, outs = L * mn;
  u64 acc[4] = {0, 0, 0, 0};
  if (o < outs) {
    const u64* w = W + o;
    const i64 step = (i64)outs;
    int p = warp, j = 0;
#pragma unroll 4
    for (; p < parts; p += 8, ++j) acc[j & 3] += __ldg(w + p * step);
  }
  red[warp][lane] = acc[0] + acc[1] + acc[2] + acc[3];
  __syncthreads();
  if (warp == 0 && o < outs) {
    const int l = o / mn, i = o - l * mn;
    u64 v = C[l * sC + i];
#pragma unroll
    for (int q = 0; q < 8; ++q) v += red[q][lane];
    Z[l * sZ + i] = v;
  }
}

// shapes mpx_beaver_tc_long takes (protocols/basic.py _long_tc mirrors this:
// the budget assumes the larger row layout for every family)
static bool long_ok(int L, int64_t M, int64_t K, int64_t N, int width) {
  return L >= 2 && L <= 3 && M >= 1 && M <= 32 && N >= 1 && N <= 32 && K >= 1 && K < (1ll << 31) && width == 64 &&
         long_smem_bytes((L * (2 * (int)M + 2 * (int)N) * LONG_RP + 127) / 128 * 128) <= 232448;
}

static int long_grid(int64_t K) {
  const int nkb = (int)((K + 31) / 32);
  // one CTA per SM; at most 512 k-blocks (16384 k) per CTA keeps the diagonals exact
  const int per = min((nkb + num_sms() - 1) / num_sms(), 512);
  return (nkb + per - 1) / per;
}

// Z [L][M][N], C [L][M][N], A [L][M][K], B [L][K][N] (party strides sZ, sC,
// sA, sB); X, Y logical M x K and K x N share views at (party, row, col)
// strides; W scratch of at least max(SMs, ceil(K / 16384)) * L * M * N words.
// M, N <= 32, 2 <= L <= 3 (all parties local), width 64.
extern "C" int mpx_beaver_tc_long(uint64_t* Z, int64_t sZ, const uint64_t* C, int64_t sC, const uint64_t* X,
                                  int64_t x_ps, int64_t x_sr, int64_t x_sc, const uint64_t* A, int64_t sA,
                                  const uint64_t* Y, int64_t y_ps, int64_t y_sr, int64_t y_sc, const uint64_t* B,
                                  int64_t sB, int L, int64_t M, int64_t K, int64_t N, int p0, int width,
                                  uint64_t* W, int64_t w_words, void* stream) {
  CHECK_ARG(Z && C && X && A && Y && B && W && p0 >= -1 && p0 < L);
  CHECK_ARG(long_ok(L, M, K, N, width));
  cudaStream_t s = (cudaStream_t)stream;
  LongArgs a;
  a.W = W;
  a.X = X;
  a.x_ps = x_ps;
  a.x_sr = x_sr;
  a.x_sc = x_sc;
  a.A = A;
  a.sA = sA;
  a.Y = Y;
  a.y_ps = y_ps;
  a.y_sr = y_sr;
  a.y_sc = y_sc;
  a.B = B;
  a.sB = sB;
  a.M = (int)M;
  a.K = (int)K;
  a.N = (int)N;
  a.p0 = p0;
  a.L = L;
  a.nkb = (int)((K + 31) / 32);
  const int grid = long_grid(K);
  CHECK_ARG(w_words >= (int64_t)grid * L * M * N);
  a.dbg = getenv("MPX_LONG_DBG") ? atoi(getenv("MPX_LONG_DBG")) : 0;
  // per-family layout: contiguous runs and 16-byte alignment allow bulk copies
  auto al16 = [](const void* p, i64 ps) { return ((uintptr_t)p & 15) == 0 && (ps & 1) == 0; };
  auto fam_mode = [&](const void* g, i64 ps, i64 sr, i64 sk, i64 R) {
    if (!al16(g, ps)) return LONG_ROW8;
    if (sr == 1 && sk == R) return LONG_KMAJ;
    if (sk == 1 && (sr & 1) == 0) return LONG_ROW16;
    return LONG_ROW8;
  };
  a.mode[0] = fam_mode(X, x_ps, x_sr, x_sc, M);
  a.mode[1] = fam_mode(A, sA, K, 1, M);
  // A_l (row-major material) by one 3D tensor-map box per 16-k half: two TMA
  // requests per block instead of one bulk copy per 256-byte row
  CUtensorMap mapA;
  memset(&mapA, 0, sizeof(mapA));
  if (a.mode[1] == LONG_ROW16 && !getenv("MPX_LONG_NO_TMAP")) {
    PFN_encodeTiled enc = get_encode();
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)M, (cuuint64_t)L};
    cuuint64_t strides[2] = {(cuuint64_t)K * 8, (cuuint64_t)sA * 8};
    cuuint32_t box[3] = {16, (cuuint32_t)M, (cuuint32_t)L};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc && enc(&mapA, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, (void*)A, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      a.mode[1] = LONG_ROWT;
  }
  a.mode[2] = fam_mode(Y, y_ps, y_sc, y_sr, N);
  a.mode[3] = fam_mode(B, sB, 1, N, N);
  if (const char* e = getenv("MPX_LONG_ROW8"))  // tests: force the generic fill
    if (atoi(e)) a.mode[0] = a.mode[1] = a.mode[2] = a.mode[3] = LONG_ROW8;
  a.tma = 1;
  a.hb = long_hb_words(L, (int)M);
  // the tensor-map family first (its half boxes need 1024-byte alignment)
  int off = 0;
  const int rows[4] = {(int)M, (int)M, (int)N, (int)N};
  const int order[4] = {1, 0, 2, 3};
  for (int f : order) {
    a.off[f] = off;
    off += long_fam_words(a.mode[f], L, rows[f]);
    off = (off + 1) & ~1;
    if (a.mode[f] == LONG_ROW8) a.tma = 0;
  }
  a.rw = (off + 127) & ~127;  // raw buffers 1024-byte aligned
  a.txb = L * (int)(2 * M + 2 * N) * 256;  // 32 words per (party, row): row pads are not copied
  const int smem = long_smem_bytes(a.rw);
  CHECK_ARG(smem <= 232448);
  static int attr[4] = {0, 0, 0, 0};
  const void* fn = L == 2 ? (const void*)k_beaver_tc_long<2> : (const void*)k_beaver_tc_long<3>;
  if (smem > attr[L]) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return MPX_ERR_CUDA;
    attr[L] = smem;
  }
  if (L == 2) k_beaver_tc_long<2><<<grid, 256, smem, s>>>(a, mapA);
  else k_beaver_tc_long<3><<<grid, 256, smem, s>>>(a, mapA);
  if (cudaGetLastError() != cudaSuccess) return MPX_ERR_CUDA;
  const int outs = L * (int)(M * N);
  k_long_reduce<<<(outs + 31) / 32, 256, 0, s>>>(Z, sZ, C, sC, W, L, (int)(M * N), grid);
  return launch_status();
}
