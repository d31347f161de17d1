// k_gemm_imad.cu — the CUDA-core 64-bit IMAD variant of the entangled integer
// matrix product: C_m = A_m B, A_m rows x K int64 (entangled),
// B K x cols int32 (the shared kernel, unmodified), C_m int64, wrap mod 2^64.
// Classic smem-tiled SIMT GEMM: CTA tile 64 x 64, K-step 16, 256 threads,
// 4 x 4 outputs per thread; the correctness anchor and the comparison point
// for the tcgen05 int8-limb kernel (k_gemm_tc.cu).
#include <cuda_runtime.h>

#include "ne_internal.cuh"

namespace ne {

constexpr int kBM = 64, kBN = 64, kBK = 16;

__global__ void __launch_bounds__(256)
k_gemm_imad64(const __grid_constant__ ne_cstreams A, const int32_t* __restrict__ B,
              const __grid_constant__ ne_streams C, int64_t rows, int64_t cols, int64_t K) {
  __shared__ int64_t As[kBK][kBM];
  __shared__ int32_t Bs[kBK][kBN];
  const int m = blockIdx.z;
  const int64_t row0 = (int64_t)blockIdx.y * kBM, col0 = (int64_t)blockIdx.x * kBN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t* __restrict__ Am = A.s[m];
  uint64_t acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;

  for (int64_t k0 = 0; k0 < K; k0 += kBK) {
    // A tile 64 x 16 (transposed into As[k][row]); B tile 16 x 64
    for (int t = threadIdx.x; t < kBM * kBK; t += 256) {
      const int r = t / kBK, kk = t % kBK;
      const int64_t gr = row0 + r, gk = k0 + kk;
      As[kk][r] = (gr < rows && gk < K) ? Am[gr * K + gk] : 0;
    }
    for (int t = threadIdx.x; t < kBK * kBN; t += 256) {
      const int kk = t / kBN, c = t % kBN;
      const int64_t gk = k0 + kk, gc = col0 + c;
      Bs[kk][c] = (gk < K && gc < cols) ? B[gk * cols + gc] : 0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      uint64_t a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = (uint64_t)As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = (uint64_t)(int64_t)Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
  int64_t* __restrict__ Cm = C.s[m];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gr = row0 + ty * 4 + i;
    if (gr >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gc = col0 + tx * 4 + j;
      if (gc < cols) Cm[gr * cols + gc] = (int64_t)acc[i][j];
    }
  }
}

void launch_gemm_imad64(int M, const ne_cstreams& A, const int32_t* B, const ne_streams& C, int64_t rows,
                        int64_t cols, int64_t K, cudaStream_t s) {
  dim3 grid((unsigned)((cols + kBN - 1) / kBN), (unsigned)((rows + kBM - 1) / kBM), (unsigned)M);
  k_gemm_imad64<<<grid, 256, 0, s>>>(A, B, C, rows, cols, K);
}

}  // namespace ne
