// Microbenchmark: HBM read bandwidth of per-warp TMA bulk-copy streams
// (cp.async.bulk + mbarrier) as a function of the copy size and the number of
// copies in flight per warp — the streaming mechanism of the sweep kernels.
// Each warp streams its own contiguous region through a shared-memory ring
// (lane 0 issues, the warp waits and touches one word per copy).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bw bulk_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b)); }
__device__ __forceinline__ void expect_tx(unsigned b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(unsigned d, const void* s, unsigned n, unsigned b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "l"(s),
               "r"(n), "r"(b) : "memory");
}
__device__ __forceinline__ void mwait(unsigned b, unsigned ph) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(b),
               "r"(ph) : "memory");
}

extern __shared__ __align__(128) unsigned char sm[];

__global__ void stream(const unsigned char* g, long long per_warp, int U, int NS, int wpb, double* sink, int fence) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long w = (long long)blockIdx.x * wpb + wib;
  unsigned char* ring = sm + (size_t)wib * (NS * U + 8 * NS);
  const unsigned bars = su32(ring + NS * U);
  if (lane == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(bars + 8 * i);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const unsigned char* src = g + w * per_warp;
  const int n = (int)(per_warp / U);
  int issued = 0;
  double acc = 0;
  for (int c = 0; c < n; ++c) {
    while (issued < n && issued - c < NS) {
      if (lane == 0) {
        const unsigned b = bars + 8 * (issued % NS);
        if (fence) asm volatile("fence.proxy.async.shared::cta;");
        expect_tx(b, U);
        bulk(su32(ring + (issued % NS) * U), src + (long long)issued * U, U, b);
      }
      ++issued;
    }
    mwait(bars + 8 * (c % NS), (c / NS) & 1);
    acc += *reinterpret_cast<const double*>(ring + (c % NS) * U + 8 * lane);
    __syncwarp();
  }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  const long long total = 8LL << 30;  // 8 GB
  unsigned char* g;
  double* sink;
  cudaMalloc(&g, total);
  cudaMalloc(&sink, 8);
  cudaMemset(g, 0, total);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  int sizes[] = {512, 1024, 2048, 4096, 8192};
  for (int fence : {1, 0})
  for (int U : sizes)
    for (int inflight_kb : {8, 16})
      for (int wps : {8, 16}) {  // warps per SM
        const int NS = inflight_kb * 1024 / U;
        if (NS < 2) continue;
        const int wpb = 4;
        const int smem = wpb * (NS * U + 8 * NS);
        if (smem * (wps / wpb) > 227 * 1024) continue;
        const long long nwarps = 148LL * wps;
        const long long per = (total / nwarps) / U * U;
        const int blocks = (int)(nwarps / wpb);
        stream<<<blocks, 32 * wpb, smem>>>(g, per, U, NS, wpb, sink, fence);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) stream<<<blocks, 32 * wpb, smem>>>(g, per, U, NS, wpb, sink, fence);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const cudaError_t e = cudaGetLastError();
        printf("fence %d copy %5d B  in-flight %2d KB/warp  warps/SM %2d : %7.0f GB/s %s\n", fence, U, inflight_kb, wps,
               3.0 * per * nwarps / (ms * 1e6), e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
