// Times k_gemm_imad32w<TM, TN> tile variants on the C3 shape (3 x 4096^3,
// entangled operand |eps| < 2^28, B in [-64, 64)).  Built once per variant:
// nvcc ... -DNE_IMAD_TM=8 -DNE_IMAD_TN=8 -I../../include -o imad_v88 imad_variants.cu
#include "../../paper_1604_04740_b200/csrc/k_gemm_imad.cu"
#include <stdio.h>

__global__ void k_fill64(int64_t* x, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z ^= z >> 29;
    x[i] = (int64_t)(z % (1ull << 28)) - (1ll << 27);
  }
}
__global__ void k_fill32(int32_t* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (int32_t)((i * 2654435761ull) % 128) - 64;
}

int main() {
  const int M = 3;
  const int64_t n = 4096;
  ne_cstreams A{};
  ne_streams C{};
  for (int m = 0; m < M; ++m) {
    int64_t *a, *c;
    cudaMalloc(&a, n * n * 8);
    cudaMalloc(&c, n * n * 8);
    k_fill64<<<1184, 256>>>(a, n * n, m);
    A.s[m] = a;
    C.s[m] = c;
  }
  int32_t* B;
  cudaMalloc(&B, n * n * 4);
  k_fill32<<<1184, 256>>>(B, n * n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ne::launch_gemm_imad32w(M, A, B, C, n, n, n, nullptr, 0);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) ne::launch_gemm_imad32w(M, A, B, C, n, n, n, nullptr, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  const double macs = (double)M * n * n * n;
  printf("TM=%d TN=%d: %.3f ms  %.2f T MAC/s  %.1f MAC/clk/SM @1965  (%s)\n", NE_IMAD_TM, NE_IMAD_TN, ms,
         macs / ms / 1e9, macs / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
