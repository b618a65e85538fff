// tcgen05 int8-limb Z_2^64 GEMM (placeholder until the tensor-core kernel lands).
#include "common.cuh"

int mpx_gemm_tc(uint64_t*, const uint64_t*, const uint64_t*, int64_t, int64_t, int64_t, int64_t, int64_t,
                int64_t, int64_t, int, int, cudaStream_t) {
  return MPX_ERR_UNSUPPORTED;
}
