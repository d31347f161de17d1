// Per-SM inbound throughput microbenchmark: each CTA streams `per` bytes from
// global memory into a 4-stage shared-memory ring with 1-D bulk copies
// (cp.async.bulk ... mbarrier::complete_tx), as a TMA producer feeding a
// consumer that only releases the stage.  All CTAs read the same 8 MB region
// (L2-resident after the first pass), or private regions (DRAM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_load(const char* src, size_t region, size_t per, int chunk, int shared_region) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t full[4];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const char* base = src + (shared_region ? 0 : (size_t)blockIdx.x * per);
  const size_t n = per / chunk;
  for (size_t i = 0; i < n + 4; ++i) {
    if (i >= 4) {  // consume chunk i-4
      const int s = (i - 4) & 3;
      const uint32_t ph = ((i - 4) >> 2) & 1;
      asm volatile(
          "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
              su32(&full[s])),
          "r"(ph));
    }
    if (i < n) {
      const int s = i & 3;
      const size_t off = (i * (size_t)chunk) % region;
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(sm + s * chunk)),
                   "l"(base + off), "r"(chunk), "r"(su32(&full[s]))
                   : "memory");
    }
  }
}

int main() {
  const size_t per = 4 << 20, region = 8 << 20;
  char* src;
  cudaMalloc(&src, 148 * per);
  cudaMemset(src, 1, 148 * per);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int chunk : {16384, 32768}) {
    cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * chunk);
    for (int shared : {1, 0})
      for (int ctas : {1, 8, 74, 148}) {
        k_load<<<ctas, 32, 4 * chunk>>>(src, shared ? region : per, per, chunk, shared);
        cudaEventRecord(a);
        k_load<<<ctas, 32, 4 * chunk>>>(src, shared ? region : per, per, chunk, shared);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("chunk=%5d %s ctas=%3d: %.1f GB/s per SM, %.0f GB/s total\n", chunk, shared ? "L2  " : "DRAM", ctas,
               per / (ms * 1e-3) / 1e9, ctas * per / (ms * 1e-3) / 1e9);
      }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
