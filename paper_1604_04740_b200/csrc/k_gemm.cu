// k_gemm.cu — ne_op_gemm dispatch (IMAD64 CUDA-core path or the tcgen05
// int8-limb path) and the operand preparation kernels of the limb path.
#include <cuda_runtime.h>

#include <climits>

#include "ne_internal.cuh"

namespace ne {

void launch_gemm_imad64(int M, const ne_cstreams& A, const int32_t* B, const ne_streams& C, int64_t rows,
                        int64_t cols, int64_t K, cudaStream_t s);
void launch_gemm_imad32w(int M, const ne_cstreams& A, const int32_t* B, const ne_streams& C, int64_t rows,
                         int64_t cols, int64_t K, ne_diag* diag, cudaStream_t s);
ne_status launch_gemm_tc(int M, int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols,
                         int64_t K, const ne_streams& C, cudaStream_t s);
void gemm_trace(long long* buf, int max_clusters);
void gemm_pair_halves(int mode);
int64_t gemm_pair_whole_tiles(int64_t n_tiles, int64_t npairs);
bool gemm_pair_gate(int M, int L, int b, int64_t rows, int64_t cols, int64_t K);
ne_status launch_gemm_tc_scatter(int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols,
                                 int64_t K, const ne_streams& dests, int ndest, int64_t* local, cudaStream_t s);
ne_status launch_gemm_tc_check(int M, int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows,
                               int64_t cols, int64_t K, const ne_streams& C, const ne_cstreams& dr,
                               const ne_streams& dor, uint32_t* bitmap, ne_diag* diag, int* cnt, int l,
                               cudaStream_t s);

// int64 entangled A_m -> L balanced int8 digit planes, planes[(m*L+i)*n + idx]
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_split_limbs(const __grid_constant__ ne_cstreams A, int M_rt, int64_t n, int L, int b, int8_t* __restrict__ planes,
              ne_diag* __restrict__ diag) {
  const int M = MT > 0 ? MT : M_rt;
  int bad = 0;
  long long first = LLONG_MAX;
  const int64_t nq = n / 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
      if (MT == 0 && m >= M) break;
      const longlong2* p = reinterpret_cast<const longlong2*>(A.s[m] + 4 * q);
      longlong2 u = __ldcs(p), w = __ldcs(p + 1);
      const int64_t x[4] = {u.x, u.y, w.x, w.y};
      uint32_t packed[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      bool ok[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int8_t d[8];
        ok[i] = digits_b(x[i], b, L, d);
        for (int j = 0; j < L; ++j) packed[j] |= (uint32_t)(uint8_t)d[j] << (8 * i);
      }
      for (int j = 0; j < L; ++j) *reinterpret_cast<uint32_t*>(planes + ((int64_t)m * L + j) * n + 4 * q) = packed[j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (!ok[i]) {
          ++bad;
          long long idx = (long long)m * n + 4 * q + i;
          first = idx < first ? idx : first;
        }
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// B (K x cols int32, row-major) -> Bt (cols x K int8, K contiguous), the
// one-plane int8 operand of the tensor-core GEMM (|B| <= 127 / -128, else a
// range violation).  Tile 64 (k) x 128 (c), 256 threads.  A task is a 4 x 4
// block (4 rows k, 4 columns c): four 128-bit loads along c, a register
// transpose into four 32-bit words (4 k-bytes of one column, PRMT), stored to
// a [128][17]-word shared tile (a warp's 8 x 4 tasks hit 32 distinct banks);
// then 128-bit stores of 16 consecutive k per column.
__global__ void __launch_bounds__(256)
k_prep_b(const int32_t* __restrict__ B, int64_t K, int64_t cols, int8_t* __restrict__ Bt, ne_diag* __restrict__ diag) {
  __shared__ uint32_t W[128][17];
  const int64_t k0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 128;
  const bool vec = (cols % 4) == 0;
  const int lane = threadIdx.x & 31;
  int bad = 0;
  long long first = LLONG_MAX;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int wt = (threadIdx.x >> 5) + 8 * it;  // 16 warp tasks of 8 (c) x 4 (k) blocks
    const int cq = (wt & 3) * 8 + (lane & 7), kq = (wt >> 2) * 4 + (lane >> 3);
    const int64_t c = c0 + 4 * cq;
    int32_t v[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t k = k0 + 4 * kq + r;
      if (k < K && vec && c + 3 < cols) {
        const int4 w = __ldcs(reinterpret_cast<const int4*>(B + k * cols + c));
        v[r][0] = w.x; v[r][1] = w.y; v[r][2] = w.z; v[r][3] = w.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[r][i] = (k < K && c + i < cols) ? B[k * cols + c + i] : 0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if ((uint32_t)(v[r][i] + 128) > 255u) {
          ++bad;
          const long long idx = (long long)((k0 + 4 * kq + r) * cols + c + i);
          first = idx < first ? idx : first;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      W[4 * cq + i][kq] = __byte_perm(__byte_perm(v[0][i], v[1][i], 0x0040), __byte_perm(v[2][i], v[3][i], 0x0040), 0x5410);
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int u = threadIdx.x + 256 * it;  // 512 chunks of 16 consecutive k
    const int cc = u >> 2, j = u & 3;
    const int64_t c = c0 + cc, k = k0 + 16 * j;
    if (c < cols && k + 15 < K)
      __stcs(reinterpret_cast<uint4*>(Bt + c * K + k), make_uint4(W[cc][4 * j], W[cc][4 * j + 1], W[cc][4 * j + 2], W[cc][4 * j + 3]));
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// B -> Bt for full tiles of 128 k x 64 columns (K % 128 == 0, cols % 64 == 0):
// each thread packs 4 consecutive k of 4 columns per task (4 x 128-bit loads,
// 16 threads per 256-byte row segment), the [64][33]-word shared tile is
// transposed so that 8 threads store one full 128-byte line of a Bt row.
// (r02 A/B, C3's 4096 x 4096 B replayed alone: 15.6 us = 5.4 TB/s; a
// persistent variant — grid of SMs x resident blocks walking the tiles, next
// tile's loads issued before this tile's stores, double-buffered shared tile —
// 18.1 us, dropped.)
__global__ void __launch_bounds__(256)
k_prep_b128(const int32_t* __restrict__ B, int64_t K, int64_t cols, int8_t* __restrict__ Bt,
            ne_diag* __restrict__ diag) {
  __shared__ uint32_t W[64][33];
  const int64_t k0 = (int64_t)blockIdx.y * 128, c0 = (int64_t)blockIdx.x * 64;
  int bad = 0;
  long long first = LLONG_MAX;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int task = it * 256 + threadIdx.x;
    const int c4 = task & 15, kq = task >> 4;  // 16 column quads x 32 k quads
    const int64_t c = c0 + 4 * c4;
    int32_t v[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t k = k0 + 4 * kq + r;
      const int4 w = __ldcs(reinterpret_cast<const int4*>(B + k * cols + c));
      v[r][0] = w.x; v[r][1] = w.y; v[r][2] = w.z; v[r][3] = w.w;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if ((uint32_t)(v[r][i] + 128) > 255u) {
          ++bad;
          const long long idx = (long long)(k * cols + c + i);
          first = idx < first ? idx : first;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      W[4 * c4 + i][kq] = __byte_perm(__byte_perm(v[0][i], v[1][i], 0x0040), __byte_perm(v[2][i], v[3][i], 0x0040), 0x5410);
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int u = it * 256 + threadIdx.x;  // 64 rows x 8 chunks of 16 bytes
    const int cc = u >> 3, j = u & 7;
    __stcs(reinterpret_cast<uint4*>(Bt + (c0 + cc) * K + k0 + 16 * j),
           make_uint4(W[cc][4 * j], W[cc][4 * j + 1], W[cc][4 * j + 2], W[cc][4 * j + 3]));
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// B (K x cols int32) -> LB balanced base-256 digit planes Bt[j][cols][K]
// (digit j = byte j of y = B + sum_{i<LB} 128 * 256^i, xor 0x80): the multi-
// plane int8 operand of a wide-range GEMM plan.  Tiles of 128 k x 64 columns
// as k_prep_b128 (K % 128 == 0, cols % 64 == 0), one [64][33]-word shared tile
// per plane; a value LB digits cannot hold is a range violation.
template <int LB>
__global__ void __launch_bounds__(256)
k_prep_b_planes(const int32_t* __restrict__ B, int64_t K, int64_t cols, int8_t* __restrict__ Bt,
                ne_diag* __restrict__ diag) {
  __shared__ uint32_t W[LB][64][33];
  constexpr int64_t bias = (int64_t)(0x8080808080808080ull >> (64 - 8 * LB));
  constexpr int64_t span = (int64_t)1 << (8 * LB);
  const int64_t k0 = (int64_t)blockIdx.y * 128, c0 = (int64_t)blockIdx.x * 64;
  int bad = 0;
  long long first = LLONG_MAX;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int task = it * 256 + threadIdx.x;
    const int c4 = task & 15, kq = task >> 4;
    const int64_t c = c0 + 4 * c4;
    int64_t y[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t k = k0 + 4 * kq + r;
      const int4 w = __ldcs(reinterpret_cast<const int4*>(B + k * cols + c));
      const int32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        y[r][i] = (int64_t)v[i] + bias;
        if (y[r][i] < 0 || y[r][i] >= span) {
          ++bad;
          const long long idx = (long long)(k * cols + c + i);
          first = idx < first ? idx : first;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < LB; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t d[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) d[r] = (uint32_t)(((y[r][i] >> (8 * j)) & 0xff) ^ 0x80);
        W[j][4 * c4 + i][kq] = d[0] | (d[1] << 8) | (d[2] << 16) | (d[3] << 24);
      }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < LB; ++j)
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int u = it * 256 + threadIdx.x;
      const int cc = u >> 3, q = u & 7;
      __stcs(reinterpret_cast<uint4*>(Bt + ((int64_t)j * cols + c0 + cc) * K + k0 + 16 * q),
             make_uint4(W[j][cc][4 * q], W[j][cc][4 * q + 1], W[j][cc][4 * q + 2], W[j][cc][4 * q + 3]));
    }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// any shape (K % 16 == 0): one thread per element, byte stores (edge shapes)
__global__ void k_prep_b_planes_any(const int32_t* __restrict__ B, int64_t K, int64_t cols, int LB,
                                    int8_t* __restrict__ Bt, ne_diag* __restrict__ diag) {
  const int64_t bias = (int64_t)(0x8080808080808080ull >> (64 - 8 * LB));
  const int64_t span = (int64_t)1 << (8 * LB);
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K * cols; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / cols, c = e % cols;
    const int64_t y = (int64_t)B[e] + bias;
    if (y < 0 || y >= span) {
      ++bad;
      first = e < first ? e : first;
    }
    for (int j = 0; j < LB; ++j) Bt[((int64_t)j * cols + c) * K + k] = (int8_t)(uint8_t)(((y >> (8 * j)) & 0xff) ^ 0x80);
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

ne_status launch_gemm_planes(int M, const int8_t* planes, int LA, const int32_t* a_shift, const int8_t* Bt, int LB,
                             int64_t rows, int64_t cols, int64_t K, const ne_streams& C, cudaStream_t s);
ne_status launch_gemm_pair_i32(int M, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols, int64_t K,
                               const ne_streams& C, cudaStream_t s);

}  // namespace ne

using namespace ne;

// balanced base-256 digits needed for |x| <= bound (digits in [-128, 127])
static int digits256(int64_t bound) {
  __int128 cap = 0, p = 1;
  for (int L = 1; L <= 8; ++L) {
    cap += 127 * p;
    p *= 256;
    if (bound <= cap) return L;
  }
  return 9;
}

extern "C" ne_status ne_gemm_plan_for(const ne_config* cfg, int64_t a_bound, int64_t b_bound, ne_gemm_plan* plan) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!plan || a_bound < 0 || b_bound < 0 || a_bound > INT32_MAX || b_bound > INT32_MAX) return NE_EINVAL;
  ne_gemm_plan p{};
  p.LB = digits256(b_bound);                 // <= 5 for |B| < 2^31
  const int l = cfg->l;
  const int Le = ne_gemm_limbs_for(cfg, a_bound);   // base-256 digits of eps = c_m + 2^l c_{m-1}
  const int D = digits256(a_bound);
  if (a_bound <= 127 && l >= 8 && l <= 31) {  // the two-digit plan: the digits are c_m and c_{m-1}
    p.kind = NE_PLAN_EPS;
    p.LA = 2;
    p.digit_bits = l;
  } else if (D <= 4 && 2 * D < Le) {          // split: c_m and c_{m-1} in D digits each, at 0 and l
    p.kind = NE_PLAN_SPLIT;
    p.LA = 2 * D;
    p.digit_bits = 8;
  } else {                                    // base-256 digits of eps
    p.kind = NE_PLAN_EPS;
    p.LA = Le;
    p.digit_bits = 8;
  }
  if (p.LA > 8) return NE_ERANGE;
  for (int i = 0; i < p.LA; ++i)
    p.a_shift[i] = p.kind == NE_PLAN_SPLIT ? (i < p.LA / 2 ? 8 * i : l + 8 * (i - p.LA / 2)) : p.digit_bits * i;
  *plan = p;
  return NE_OK;
}

extern "C" ne_status ne_gemm_prep_b_planes(const int32_t* B, int64_t K, int64_t cols, int32_t LB, int8_t* Bt,
                                           ne_diag* diag, ne_stream_t stream) {
  if (!B || !Bt || K <= 0 || cols <= 0 || K % 16 != 0 || LB < 1 || LB > 5 || !aligned16(Bt) || !aligned16(B))
    return NE_EINVAL;
  cudaStream_t s = cs(stream);
  if (K % 128 == 0 && cols % 64 == 0) {
    const dim3 grid((unsigned)(cols / 64), (unsigned)(K / 128));
    switch (LB) {
      case 1: k_prep_b_planes<1><<<grid, 256, 0, s>>>(B, K, cols, Bt, diag); break;
      case 2: k_prep_b_planes<2><<<grid, 256, 0, s>>>(B, K, cols, Bt, diag); break;
      case 3: k_prep_b_planes<3><<<grid, 256, 0, s>>>(B, K, cols, Bt, diag); break;
      case 4: k_prep_b_planes<4><<<grid, 256, 0, s>>>(B, K, cols, Bt, diag); break;
      default: k_prep_b_planes<5><<<grid, 256, 0, s>>>(B, K, cols, Bt, diag); break;
    }
    return launch_status();
  }
  k_prep_b_planes_any<<<grid_for(K * cols, 256), 256, 0, s>>>(B, K, cols, LB, Bt, diag);
  return launch_status();
}

static bool tc_shape_ok(int64_t rows, int64_t cols, int64_t K) {
  return rows > 0 && cols > 0 && K > 0 && rows % 128 == 0 && cols % 128 == 0 && K % 128 == 0 && K < 131072;  // K * 2^14 < 2^31
}

extern "C" ne_status ne_gemm_workspace(const ne_config* cfg, int64_t rows, int64_t cols, int64_t K, int32_t L,
                                       int32_t LB, size_t* bytes) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!bytes || L < 1 || L > 8 || LB < 1 || LB > 5) return NE_EINVAL;
  *bytes = (size_t)cfg->M * L * rows * K + (size_t)LB * cols * K + 1024;
  return NE_OK;
}

extern "C" ne_status ne_gemm_prep_b(const int32_t* B, int64_t K, int64_t cols, int8_t* Bt, ne_diag* diag,
                                    ne_stream_t stream) {
  if (!B || !Bt || K <= 0 || cols <= 0 || K % 16 != 0 || !aligned16(Bt) || !aligned16(B)) return NE_EINVAL;
  if (K % 128 == 0 && cols % 64 == 0) {
    k_prep_b128<<<dim3((unsigned)(cols / 64), (unsigned)(K / 128)), 256, 0, cs(stream)>>>(B, K, cols, Bt, diag);
    return launch_status();
  }
  dim3 grid((unsigned)((cols + 127) / 128), (unsigned)((K + 63) / 64));
  k_prep_b<<<grid, 256, 0, cs(stream)>>>(B, K, cols, Bt, diag);
  return launch_status();
}

extern "C" ne_status ne_op_gemm_limbs(const ne_config* cfg, const int8_t* planes, int32_t L, int32_t limb_bits,
                                      const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, ne_streams C,
                                      ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!planes || !Bt || L < 1 || L > 4 || limb_bits < 8 || limb_bits > 63 || !aligned16(planes) || !aligned16(Bt))
    return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (!C.s[m] || !aligned16(C.s[m])) return NE_EINVAL;
  if (!tc_shape_ok(rows, cols, K)) return NE_ENOTSUP;
  return launch_gemm_tc(cfg->M, L, limb_bits, planes, Bt, rows, cols, K, C, cs(stream));
}

extern "C" ne_status ne_op_gemm_plan(const ne_config* cfg, const int8_t* planes, const ne_gemm_plan* plan,
                                     const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, ne_streams C,
                                     ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!plan || !planes || !Bt || plan->LA < 1 || plan->LA > 8 || plan->LB < 1 || plan->LB > 5 ||
      !aligned16(planes) || !aligned16(Bt))
    return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (!C.s[m] || !aligned16(C.s[m])) return NE_EINVAL;
  if (!tc_shape_ok(rows, cols, K)) return NE_ENOTSUP;
  return launch_gemm_planes(cfg->M, planes, plan->LA, plan->a_shift, Bt, plan->LB, rows, cols, K, C, cs(stream));
}

extern "C" ne_status ne_op_gemm_plain_i32(int32_t count, const int8_t* planes, const int8_t* Bt, int64_t rows,
                                          int64_t cols, int64_t K, ne_streams32 C, ne_stream_t stream) {
  if (count < 1 || count > 8 || !planes || !Bt || !aligned16(planes) || !aligned16(Bt)) return NE_EINVAL;
  for (int m = 0; m < count; ++m)
    if (!C.s[m] || !aligned16(C.s[m])) return NE_EINVAL;
  if (!tc_shape_ok(rows, cols, K) || rows % 256 || cols % 256) return NE_ENOTSUP;
  ne_streams Cs{};
  for (int m = 0; m < count; ++m) Cs.s[m] = reinterpret_cast<int64_t*>(C.s[m]);
  return launch_gemm_pair_i32(count, planes, Bt, rows, cols, K, Cs, cs(stream));
}

extern "C" ne_status ne_gemm_kernel_for(const ne_config* cfg, int32_t L, int32_t limb_bits, int64_t rows,
                                        int64_t cols, int64_t K, int32_t* kernel) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!kernel || L < 1 || L > 4 || limb_bits < 8 || limb_bits > 63) return NE_EINVAL;
  if (!tc_shape_ok(rows, cols, K)) return NE_ENOTSUP;
  *kernel = gemm_pair_gate(cfg->M, L, limb_bits, rows, cols, K) ? NE_GEMM_KERNEL_PAIR : NE_GEMM_KERNEL_CTA;
  return NE_OK;
}

extern "C" ne_status ne_gemm_trace(long long* buf, int32_t max_clusters) {
  if (max_clusters < 0) return NE_EINVAL;
  gemm_trace(buf, max_clusters);
  return NE_OK;
}

extern "C" ne_status ne_gemm_pair_halves(int32_t mode) {
  if (mode < 0 || mode > 2) return NE_EINVAL;
  gemm_pair_halves(mode);
  return NE_OK;
}

extern "C" ne_status ne_gemm_pair_schedule(int64_t n_tiles, int64_t npairs, int64_t* n_whole) {
  if (!n_whole || n_tiles < 0 || npairs < 1) return NE_EINVAL;
  *n_whole = gemm_pair_whole_tiles(n_tiles, npairs);
  return NE_OK;
}

extern "C" ne_status ne_gemm_check_workspace(int64_t rows, int64_t cols, size_t* bytes) {
  if (!bytes || rows < 0 || cols < 0) return NE_EINVAL;
  *bytes = (size_t)((rows + 127) / 128) * (size_t)((cols + 127) / 128) * sizeof(int32_t) + 16;
  return NE_OK;
}

extern "C" ne_status ne_op_gemm_limbs_check(const ne_config* cfg, const int8_t* planes, int32_t L, int32_t limb_bits,
                                            const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, ne_streams C,
                                            int32_t r, ne_streams d_out, uint32_t* bitmap, ne_diag* diag,
                                            int32_t* tile_counters, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  if (!planes || !Bt || !tile_counters || L < 1 || L > 4 || limb_bits < 8 || limb_bits > 63 || !aligned16(planes) ||
      !aligned16(Bt))
    return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (!C.s[m] || !aligned16(C.s[m]) || !d_out.s[m] || !aligned16(d_out.s[m])) return NE_EINVAL;
  if (!tc_shape_ok(rows, cols, K)) return NE_ENOTSUP;
  cudaStream_t s = cs(stream);
  ne_cstreams Cc{};
  for (int m = 0; m < cfg->M; ++m) Cc.s[m] = C.s[m];
  st = launch_gemm_tc_check(cfg->M, L, limb_bits, planes, Bt, rows, cols, K, C, rotate(Cc, cfg->M, r),
                            rotate(d_out, cfg->M, r), bitmap, diag, tile_counters, cfg->l, s);
  if (st != NE_ENOTSUP) return st;
  if ((st = launch_gemm_tc(cfg->M, L, limb_bits, planes, Bt, rows, cols, K, C, s)) != NE_OK) return st;
  return ne_disentangle_check(cfg, Cc, rows * cols, r, d_out, bitmap, diag, stream);
}

extern "C" ne_status ne_op_gemm_limbs_stream(const ne_config* cfg, const int8_t* planes_m, int32_t L,
                                             int32_t limb_bits, const int8_t* Bt, int64_t rows, int64_t cols,
                                             int64_t K, int64_t* C_m, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!planes_m || !Bt || !C_m || L < 1 || L > 4 || limb_bits < 8 || limb_bits > 63 || !aligned16(planes_m) ||
      !aligned16(Bt) || !aligned16(C_m))
    return NE_EINVAL;
  if (!tc_shape_ok(rows, cols, K)) return NE_ENOTSUP;
  ne_streams C{};
  C.s[0] = C_m;
  return launch_gemm_tc(1, L, limb_bits, planes_m, Bt, rows, cols, K, C, cs(stream));
}

extern "C" ne_status ne_op_gemm_limbs_scatter(const ne_config* cfg, const int8_t* planes_m, int32_t L,
                                              int32_t limb_bits, const int8_t* Bt, int64_t rows, int64_t cols,
                                              int64_t K, ne_streams dests, int32_t ndest, int64_t* C_local,
                                              ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!planes_m || !Bt || L < 1 || L > 4 || limb_bits < 8 || limb_bits > 63 || !aligned16(planes_m) ||
      !aligned16(Bt) || ndest < 1 || ndest > 8)
    return NE_EINVAL;
  for (int j = 0; j < ndest; ++j)
    if (!dests.s[j] || !aligned16(dests.s[j])) return NE_EINVAL;
  if (C_local && !aligned16(C_local)) return NE_EINVAL;
  if (!tc_shape_ok(rows, cols, K) || rows % (128 * (int64_t)ndest) != 0) return NE_ENOTSUP;
  return launch_gemm_tc_scatter(L, limb_bits, planes_m, Bt, rows, cols, K, dests, ndest, C_local, cs(stream));
}

extern "C" ne_status ne_op_gemm(const ne_config* cfg, ne_cstreams A, const int32_t* B, int64_t rows, int64_t cols,
                                int64_t K, ne_gemm_algo algo, int32_t L, int32_t limb_bits, int32_t LB, ne_streams C,
                                void* ws, size_t ws_bytes, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  const int M = cfg->M;
  if (!B || rows < 0 || cols < 0 || K < 0) return NE_EINVAL;
  for (int m = 0; m < M; ++m)
    if (!A.s[m] || !C.s[m] || !aligned16(A.s[m]) || !aligned16(C.s[m])) return NE_EINVAL;
  if (rows == 0 || cols == 0) return NE_OK;
  cudaStream_t s = cs(stream);
  if (algo == NE_GEMM_IMAD64) {
    launch_gemm_imad64(M, A, B, C, rows, cols, K, s);
    return launch_status();
  }
  if (algo == NE_GEMM_IMAD32W) {
    if (rows % 128 || cols % 128 || K % 16 || K == 0) {  // tile-aligned shapes only: the any-shape 64-bit form
      launch_gemm_imad64(M, A, B, C, rows, cols, K, s);
      return launch_status();
    }
    if (!aligned16(B)) return NE_EINVAL;
    launch_gemm_imad32w(M, A, B, C, rows, cols, K, diag, s);
    return launch_status();
  }
  if (algo != NE_GEMM_TC_I8) return NE_EINVAL;
  if (L < 1 || L > 8 || LB < 1 || LB > 5 || limb_bits < 8 || limb_bits > 63 || limb_bits * (L - 1) > 63)
    return NE_EINVAL;
  if (!tc_shape_ok(rows, cols, K)) return NE_ENOTSUP;
  size_t need = 0;
  ne_gemm_workspace(cfg, rows, cols, K, L, LB, &need);
  if (!ws || ws_bytes < need || !aligned16(ws)) return NE_EINVAL;
  int8_t* planes = static_cast<int8_t*>(ws);
  int8_t* Bt = planes + (size_t)M * L * rows * K;
  const int64_t n = rows * K;
  const int grid = grid_for(n / 4, kThreads);
  switch (M) {
    case 3: k_split_limbs<3><<<grid, kThreads, 0, s>>>(A, 3, n, L, limb_bits, planes, diag); break;
    case 4: k_split_limbs<4><<<grid, kThreads, 0, s>>>(A, 4, n, L, limb_bits, planes, diag); break;
    case 8: k_split_limbs<8><<<grid, kThreads, 0, s>>>(A, 8, n, L, limb_bits, planes, diag); break;
    default: k_split_limbs<0><<<grid, kThreads, 0, s>>>(A, M, n, L, limb_bits, planes, diag); break;
  }
  if ((st = launch_status()) != NE_OK) return st;
  if (LB == 1) {
    if ((st = ne_gemm_prep_b(B, K, cols, Bt, diag, stream)) != NE_OK) return st;
    if (L <= 4) return launch_gemm_tc(M, L, limb_bits, planes, Bt, rows, cols, K, C, s);
  } else if ((st = ne_gemm_prep_b_planes(B, K, cols, LB, Bt, diag, stream)) != NE_OK) {
    return st;
  }
  int32_t sh[8];
  for (int i = 0; i < L; ++i) sh[i] = limb_bits * i;
  return launch_gemm_planes(M, planes, L, sh, Bt, LB, rows, cols, K, C, s);
}
