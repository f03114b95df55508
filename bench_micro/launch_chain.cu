// Launch-boundary cost on B200: a CUDA graph of N dependent tiny kernels
// (with / without programmatic dependent launch) against one persistent
// kernel with N software grid barriers.  Informs whether fusing the Krylov
// iteration's ~27 latency-bound launches into one persistent kernel pays.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(double* a, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  a[i] = a[i] * 1.0000001 + 1.0;
}

__device__ unsigned int g_bar;
__global__ void k_persist(double* a, int n, unsigned int base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < n; ++k) {
    a[i] = a[i] * 1.0000001 + 1.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned int target = base + (unsigned int)(k + 1) * gridDim.x;
      atomicAdd(&g_bar, 1u);
      while (*(volatile unsigned int*)&g_bar < target) {
      }
      __threadfence();
    }
    __syncthreads();
  }
}

int main() {
  const int N = 30, blocks = 148 * 2, threads = 128;
  double* a;
  cudaMalloc(&a, sizeof(double) * blocks * threads);
  cudaMemset(a, 0, sizeof(double) * blocks * threads);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < N; ++k) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = blocks, cfg.blockDim = threads, cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at, cfg.numAttrs = pdl;
      cudaLaunchKernelEx(&cfg, k_tiny, a, pdl);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < 100; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("graph of %d tiny kernels (pdl=%d): %.2f us per kernel\n", N, pdl, ms * 1e3 / (100 * N));
  }
  unsigned int base = 0;
  cudaMemcpyToSymbol(g_bar, &base, sizeof base);
  for (int w = 0; w < 5; ++w, base += N * blocks) k_persist<<<blocks, threads, 0, st>>>(a, N, base);
  cudaEventRecord(e0, st);
  for (int r = 0; r < 100; ++r, base += N * blocks) k_persist<<<blocks, threads, 0, st>>>(a, N, base);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("persistent kernel, %d grid barriers (%d CTAs): %.2f us per phase\n", N, blocks, ms * 1e3 / (100 * N));
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
