// k_gemm_imad.cu — the CUDA-core 64-bit IMAD variant of the entangled integer
// matrix product: C_m = A_m B, A_m rows x K int64 (entangled),
// B K x cols int32 (the shared kernel, unmodified), C_m int64, wrap mod 2^64.
// Classic smem-tiled SIMT GEMM: CTA tile 64 x 64, K-step 16, 256 threads,
// 4 x 4 outputs per thread; the correctness anchor and the comparison point
// for the tcgen05 int8-limb kernel (k_gemm_tc.cu).
#include <cuda_runtime.h>

#include <climits>

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

// 32 x 32 -> 64-bit form (NE_GEMM_IMAD32W): when every entangled A entry
// fits int32 (the C3 operand: |eps| <= 64 (2^22 + 1) < 2^31) each MAC is one
// IMAD.WIDE (mad.wide.s32: 32 x 32 -> 64-bit product + 64-bit accumulator,
// wrap mod 2^64 — the same value as the int64 form).  CTA tile 128 x 128,
// K-step 16, 256 threads, 8 x 8 outputs per thread in two 4-row x two
// 4-column quadrants (conflict-free 128-bit shared loads), the next K-step's
// global loads in registers while the current one is multiplied.  rows and
// cols multiples of 128, K of 16 (else the IMAD64 kernel runs).  An A entry
// outside int32 is a range violation (diag), its product undefined.
constexpr int kWK = 16;
#ifndef NE_IMAD_KUNROLL
#define NE_IMAD_KUNROLL 16
#endif
constexpr int kKUnroll = NE_IMAD_KUNROLL;

__device__ __forceinline__ int64_t mad_wide(int32_t a, int32_t b, int64_t c) {
  int64_t d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

// TM x TN outputs per thread (two TM/2-row x two TN/2-column quadrants of the
// CTA tile 16 TM x 16 TN), 256 threads
template <int TM, int TN>
__global__ void __launch_bounds__(256)
k_gemm_imad32w(const __grid_constant__ ne_cstreams A, const int32_t* __restrict__ B,
               const __grid_constant__ ne_streams C, int64_t rows, int64_t cols, int64_t K,
               ne_diag* __restrict__ diag) {
  constexpr int BMc = 16 * TM, BNc = 16 * TN, HM = TM / 2, HN = TN / 2;
  // A is stored transposed (k-major): a row pad of 4 int32 spreads a warp's
  // 16 k-rows over 8 banks (2-way) instead of one (16-way: ncu counted 755 M
  // shared-store bank conflicts per C3 launch), keeping 16-B aligned rows for
  // the 128-bit reads
  __shared__ __align__(16) int32_t As[2][kWK][BMc + 4];
  __shared__ __align__(16) int32_t Bs[2][kWK][BNc];
  const int m = blockIdx.z;
  const int64_t row0 = (int64_t)blockIdx.y * BMc, col0 = (int64_t)blockIdx.x * BNc;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t* __restrict__ Am = A.s[m];
  int bad = 0;
  long long first = LLONG_MAX;
  // A entry u (u < TM): row tid / 16 + 16 u, k tid % 16; B entry u (u < TN): k tid / BNc + (256 / BNc) u,
  // col tid % BNc (rows, cols multiples of the tile and K of 16: no bounds checks)
  const int64_t* pa = Am + (row0 + (threadIdx.x >> 4)) * K + (threadIdx.x & 15);
  const int32_t* pb = B + (int64_t)(threadIdx.x / BNc) * cols + col0 + (threadIdx.x % BNc);
  int32_t ra[TM], rb[TN];
  auto load = [&](int64_t k0) {
    uint32_t badm = 0;
#pragma unroll
    for (int u = 0; u < TM; ++u) {
      const int64_t x = __ldg(pa + 16 * u * K + k0);
      ra[u] = (int32_t)x;
      badm |= (uint32_t)(x != (int64_t)ra[u]) << u;
    }
#pragma unroll
    for (int u = 0; u < TN; ++u) rb[u] = __ldg(pb + (k0 + (256 / BNc) * u) * cols);
    if (badm) {  // an entry outside int32: range violation naming m * rows * K + row * K + k
      for (int u = 0; u < TM; ++u)
        if (badm >> u & 1) {
          ++bad;
          const long long idx = ((long long)m * rows + row0 + (threadIdx.x >> 4) + 16 * u) * K + k0 + (threadIdx.x & 15);
          first = idx < first ? idx : first;
        }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < TM; ++u) {
      const int t = threadIdx.x + 256 * u;
      As[buf][t & 15][t >> 4] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < TN; ++u) {
      const int t = threadIdx.x + 256 * u;
      Bs[buf][t / BNc][t % BNc] = rb[u];
    }
  };
  int64_t acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0;
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < K; k0 += kWK) {
    const bool more = k0 + kWK < K;
    if (more) load(k0 + kWK);
    // (fully unrolled: ptxas pairs two products of one accumulator into
    // IMAD.WIDE x 2 + a 3-input 64-bit add; one k per iteration keeps pure
    // IMAD.WIDE chains but measured slower: 16.4 vs 19.0 MAC/clk/SM)
#pragma unroll kKUnroll
    for (int kk = 0; kk < kWK; ++kk) {
      int32_t a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < HM; ++i) {
        a[i] = As[buf][kk][ty * HM + i];
        a[HM + i] = As[buf][kk][BMc / 2 + ty * HM + i];
      }
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        b[j] = Bs[buf][kk][tx * HN + j];
        b[HN + j] = Bs[buf][kk][BNc / 2 + tx * HN + j];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = mad_wide(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  int64_t* __restrict__ Cm = C.s[m];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t gr = row0 + (i < HM ? ty * HM + i : BMc / 2 + ty * HM + i - HM);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t gc = col0 + h * (BNc / 2) + tx * HN;
#pragma unroll
      for (int j = 0; j < HN; j += 2)
        *reinterpret_cast<longlong2*>(Cm + gr * cols + gc + j) = make_longlong2(acc[i][h * HN + j], acc[i][h * HN + j + 1]);
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

#ifndef NE_IMAD_TM
#define NE_IMAD_TM 8
#endif
#ifndef NE_IMAD_TN
#define NE_IMAD_TN 8
#endif
constexpr int kWM = 16 * NE_IMAD_TM, kWN = 16 * NE_IMAD_TN;

void launch_gemm_imad32w(int M, const ne_cstreams& A, const int32_t* B, const ne_streams& C, int64_t rows,
                         int64_t cols, int64_t K, ne_diag* diag, cudaStream_t s) {
  dim3 grid((unsigned)(cols / kWN), (unsigned)(rows / kWM), (unsigned)M);
  k_gemm_imad32w<NE_IMAD_TM, NE_IMAD_TN><<<grid, 256, 0, s>>>(A, B, C, rows, cols, K, diag);
}

void launch_gemm_imad64(int M, const ne_cstreams& A, const int32_t* B, const ne_streams& C, int64_t rows,
                        int64_t cols, int64_t K, cudaStream_t s) {
  dim3 grid((unsigned)((cols + kBN - 1) / kBN), (unsigned)((rows + kBM - 1) / kBM), (unsigned)M);
  k_gemm_imad64<<<grid, 256, 0, s>>>(A, B, C, rows, cols, K);
}

}  // namespace ne
