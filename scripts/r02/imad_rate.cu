// Issue rate of the integer multiply-adds on B200 CUDA cores: IMAD (32-bit),
// IMAD.WIDE (32 x 32 + 64 -> 64), per SM per clock, 16 independent
// accumulator chains per thread.  The multiplier changes every iteration
// (an xorshift on the ALU pipe) so the products cannot be hoisted out of the
// loop (the first version of this benchmark let ptxas do exactly that).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imad_rate imad_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int KIND>
__global__ void __launch_bounds__(256) k_rate(int iters, int32_t a, int32_t b, int64_t* out) {
  int64_t acc[16];
  int32_t acc32[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc[i] = threadIdx.x + i; acc32[i] = threadIdx.x + i; }
  uint32_t r = a + threadIdx.x * 2654435761u + blockIdx.x;
  const int32_t y = b ^ blockIdx.x;
  for (int it = 0; it < iters; ++it) {
    r ^= r << 13;
    r ^= r >> 17;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int32_t x = (int32_t)(r + i);
      if (KIND == 0) {
        asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(acc32[i]) : "r"(x), "r"(y));
      } else {
        asm volatile("mad.wide.s32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(x), "r"(y));
      }
    }
  }
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i] + acc32[i];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

int main() {
  int nsm = 148, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int grid = nsm * 8, iters = 1 << 14;
  int64_t* out;
  cudaMalloc(&out, (size_t)grid * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int kind = 0; kind < 2; ++kind) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k_rate<0><<<grid, 256>>>(iters, 3, 5, out); else k_rate<1><<<grid, 256>>>(iters, 3, 5, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)grid * 256 * iters * 16;
      if (rep)
        printf("%-10s %.3f ms  %.2f T op/s  = %.1f lane-ops/clk/SM at the %d MHz attribute clock\n",
               kind ? "IMAD.WIDE" : "IMAD", ms, ops / ms / 1e9, ops / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
