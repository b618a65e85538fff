// Philox4x64-10 ALU ceiling on one B200: blocks/s for 1/2/4 independent
// blocks per thread (ILP) and two multiply formulations. No memory traffic
// besides one XOR-folded word per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o philox_bench philox_bench.cu
#include <cstdint>
#include <cstdio>
typedef uint64_t u64;

__device__ __forceinline__ void mulhilo_c(u64 x, u64 m, u64& lo, u64& hi) {
  lo = m * x;
  hi = __umul64hi(m, x);
}

// 64x64 -> 128 from four 32x32 -> 64 IMAD.WIDE (explicit carry chain)
__device__ __forceinline__ void mulhilo_w(u64 x, u64 m, u64& lo, u64& hi) {
  const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32);
  const uint32_t m0 = (uint32_t)m, m1 = (uint32_t)(m >> 32);
  const u64 p = (u64)x0 * m0;
  const u64 q = (u64)x0 * m1 + (p >> 32);
  const u64 r = (u64)x1 * m0 + (uint32_t)q;
  lo = (r << 32) | (uint32_t)p;
  hi = (u64)x1 * m1 + (q >> 32) + (r >> 32);
}

template <int V>
__device__ __forceinline__ void round10(u64 (&c)[4], u64 k0, u64 k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    u64 lo0, hi0, lo1, hi1;
    if (V == 0) {
      mulhilo_c(c[0], 0xD2E7470EE14C6C93ull, lo0, hi0);
      mulhilo_c(c[2], 0xCA5A826395121157ull, lo1, hi1);
    } else {
      mulhilo_w(c[0], 0xD2E7470EE14C6C93ull, lo0, hi0);
      mulhilo_w(c[2], 0xCA5A826395121157ull, lo1, hi1);
    }
    const u64 n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
}

template <int V, int ILP>
__global__ void __launch_bounds__(256) k_bench(u64* out, u64 k0, u64 k1, long blocks) {
  u64 acc = 0;
  const long stride = (long)gridDim.x * blockDim.x * ILP;
  for (long b = ((long)blockIdx.x * blockDim.x + threadIdx.x) * ILP; b < blocks; b += stride) {
    u64 c[ILP][4];
#pragma unroll
    for (int j = 0; j < ILP; ++j) { c[j][0] = b + j + 1; c[j][1] = c[j][2] = c[j][3] = 0; }
#pragma unroll
    for (int j = 0; j < ILP; ++j) round10<V>(c[j], k0, k1);
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc ^= c[j][0] ^ c[j][1] ^ c[j][2] ^ c[j][3];
  }
  out[(long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V, int ILP>
void run(const char* name, u64* out, int grid, long blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 2; ++i) k_bench<V, ILP><<<grid, 256>>>(out, 1, 2, blocks);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k_bench<V, ILP><<<grid, 256>>>(out, 1, 2, blocks);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("{\"variant\": \"%s\", \"grid\": %d, \"ms\": %.3f, \"Gblocks_per_s\": %.2f, \"stream_GBps\": %.1f}\n", name,
         grid, ms, blocks / ms / 1e6, blocks * 32.0 / ms / 1e6);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long blocks = 1L << 28;
  u64* out;
  cudaMalloc(&out, sizeof(u64) * 256L * sms * 64);
  for (int occ : {4, 8, 16}) {
    const int grid = sms * occ;
    run<0, 1>("umul64hi ILP1", out, grid, blocks);
    run<0, 2>("umul64hi ILP2", out, grid, blocks);
    run<0, 4>("umul64hi ILP4", out, grid, blocks);
    run<1, 1>("wide ILP1", out, grid, blocks);
    run<1, 2>("wide ILP2", out, grid, blocks);
    run<1, 4>("wide ILP4", out, grid, blocks);
  }
  return 0;
}
