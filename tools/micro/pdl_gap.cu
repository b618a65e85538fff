// Graph launch gap between dependent small kernels, with and without
// programmatic dependent launch (PDL). nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_gap.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(unsigned long long* buf, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = buf[i] * 3 + 1;
}

int main() {
  const int n = 148 * 256, iters = 200;
  unsigned long long* buf;
  cudaMalloc(&buf, n * 8);
  cudaMemset(buf, 0, n * 8);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < iters; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, k_step, buf, n, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d: %.3f us per kernel (graph of %d)\n", pdl, ms * 1e3 / (10 * iters), iters);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
