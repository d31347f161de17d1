// k_abft.cu — the paper's comparison method on the same hardware: single-
// checksum ABFT (Eqs. 3-6).  Streaming kernels (HBM-bound):
//   encode  r_n = sum_m c_{m,n}                      (Eq. 4)
//   check   flag_n = [sum_m d_{m,n} != e_n]          (Eq. 6), mod 2^64
//   recover d_r = e - sum_{m != r} d_m
// plus the plain-data digit planes the tensor-core GEMM consumes.
#include <cuda_runtime.h>

#include <climits>

#include "ne_internal.cuh"

namespace ne {

__global__ void __launch_bounds__(kThreads)
k_abft_encode(const __grid_constant__ ne_cstreams32 c, int M, int64_t n, int32_t* __restrict__ r,
              ne_diag* __restrict__ diag) {
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < (n + 3) / 4;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    int64_t acc[4] = {0, 0, 0, 0};
    if (n0 + 4 <= n) {
      for (int m = 0; m < M; ++m) {
        const int4 q = __ldcs(reinterpret_cast<const int4*>(c.s[m] + n0));
        acc[0] += q.x; acc[1] += q.y; acc[2] += q.z; acc[3] += q.w;
      }
    } else {
      for (int m = 0; m < M; ++m)
        for (int i = 0; i < 4; ++i)
          if (n0 + i < n) acc[i] += c.s[m][n0 + i];
    }
    for (int i = 0; i < 4 && n0 + i < n; ++i) {
      if (acc[i] != (int64_t)(int32_t)acc[i]) {  // the checksum's extra log2(M) bits overflow int32
        ++bad;
        first = (n0 + i) < first ? (n0 + i) : first;
      }
      r[n0 + i] = (int32_t)acc[i];
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// plain int32 streams -> L balanced int8 digit planes (same digit trick as k_entangle_limbs)
template <int L>
__global__ void __launch_bounds__(kThreads)
k_to_limbs(const __grid_constant__ ne_cstreams32 x, int count, int64_t n, int8_t* __restrict__ planes,
           ne_diag* __restrict__ diag) {
  constexpr uint64_t bias = 0x8080808080808080ull >> (64 - 8 * L);
  constexpr uint64_t span = L == 8 ? 0 : (1ull << (8 * L));
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n / 4; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    for (int s = 0; s < count; ++s) {
      const int4 q = __ldcs(reinterpret_cast<const int4*>(x.s[s] + n0));
      const int32_t cc[4] = {q.x, q.y, q.z, q.w};
      uint64_t y[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        y[i] = (uint64_t)(int64_t)cc[i] + bias;
        if (L < 8 && y[i] >= span) {
          ++bad;
          const long long idx = (long long)s * n + n0 + i;
          first = idx < first ? idx : first;
        }
      }
#pragma unroll
      for (int j = 0; j < L; ++j) {
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) w |= (uint32_t)((y[i] >> (8 * j)) & 0xff) << (8 * i);
        __stcs(reinterpret_cast<unsigned int*>(planes + ((int64_t)s * L + j) * n + n0), w ^ 0x80808080u);
      }
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// encode + digit planes in one pass (the tensor-core form of Eqs. 4-5):
// data planes[m*n + idx] = c_m (1 int8 digit), sum planes[j*n + idx] = digit j
// of r = sum_m c_m in base 256 (LS digits).  Values that do not fit are range
// violations naming m*n + idx (data) or M*n + idx (checksum).
template <int MT, int LS>
__global__ void __launch_bounds__(kThreads)
k_abft_encode_limbs(const __grid_constant__ ne_cstreams32 c, int M_rt, int64_t n, int8_t* __restrict__ pdata,
                    int8_t* __restrict__ psum, ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  constexpr uint64_t bias = 0x8080808080808080ull >> (64 - 8 * LS);
  constexpr uint64_t span = LS == 8 ? 0 : (1ull << (8 * LS));
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n / 4; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    int4 q[MA];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) q[m] = __ldcs(reinterpret_cast<const int4*>(c.s[m] + n0));
    int64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      const int32_t cc[4] = {q[m].x, q[m].y, q[m].z, q[m].w};
      uint32_t w = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i] += cc[i];
        if (cc[i] < -128 || cc[i] > 127) {
          ++bad;
          const long long idx = (long long)m * n + n0 + i;
          first = idx < first ? idx : first;
        }
        w |= (uint32_t)(uint8_t)(int8_t)cc[i] << (8 * i);
      }
      __stcs(reinterpret_cast<unsigned int*>(pdata + (int64_t)m * n + n0), w);
    }
    uint32_t ws[LS];
#pragma unroll
    for (int j = 0; j < LS; ++j) ws[j] = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t y = (uint64_t)acc[i] + bias;
      if (LS < 8 && y >= span) {
        ++bad;
        const long long idx = (long long)M * n + n0 + i;
        first = idx < first ? idx : first;
      }
#pragma unroll
      for (int j = 0; j < LS; ++j) ws[j] |= (uint32_t)(((y >> (8 * j)) & 0xff) ^ 0x80) << (8 * i);
    }
#pragma unroll
    for (int j = 0; j < LS; ++j) __stcs(reinterpret_cast<unsigned int*>(psum + (int64_t)j * n + n0), ws[j]);
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

__device__ __forceinline__ uint32_t spread16b(uint32_t x) {
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// check: two positions per thread (128-bit loads), bitmap words from ballots
__global__ void __launch_bounds__(kThreads)
k_abft_check(const __grid_constant__ ne_cstreams d, int M, const int64_t* __restrict__ e, int64_t n,
             uint32_t* __restrict__ bitmap, ne_diag* __restrict__ diag) {
  const int lane = threadIdx.x & 31;
  const int64_t npair = (n + 1) / 2, nwords = (n + 31) / 32;
  const int64_t npair_w = (npair + 31) & ~(int64_t)31;
  int nflag = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < npair_w; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 2 * v;
    bool f0 = false, f1 = false;
    if (n0 < n) {
      const bool pair = n0 + 1 < n;
      uint64_t s0 = 0, s1 = 0;
      for (int m = 0; m < M; ++m) {
        if (pair) {
          const longlong2 q = __ldcs(reinterpret_cast<const longlong2*>(d.s[m] + n0));
          s0 += (uint64_t)q.x;
          s1 += (uint64_t)q.y;
        } else {
          s0 += (uint64_t)d.s[m][n0];
        }
      }
      if (pair) {
        const longlong2 q = __ldcs(reinterpret_cast<const longlong2*>(e + n0));
        f0 = s0 != (uint64_t)q.x;
        f1 = s1 != (uint64_t)q.y;
      } else {
        f0 = s0 != (uint64_t)e[n0];
      }
      if (f0) { ++nflag; first = n0 < first ? n0 : first; }
      if (f1) { ++nflag; first = (n0 + 1) < first ? (n0 + 1) : first; }
    }
    if (bitmap) {
      const uint32_t b0 = __ballot_sync(0xffffffffu, f0), b1 = __ballot_sync(0xffffffffu, f1);
      const int64_t w0 = (v - lane) / 16;
      if (lane == 0 && w0 < nwords) bitmap[w0] = spread16b(b0) | (spread16b(b1) << 1);
      if (lane == 1 && w0 + 1 < nwords) bitmap[w0 + 1] = spread16b(b0 >> 16) | (spread16b(b1 >> 16) << 1);
    }
  }
  if (diag) diag_add(&diag->fault_positions, &diag->first_fault, nflag, first);
}

__global__ void __launch_bounds__(kThreads)
k_abft_recover(const __grid_constant__ ne_cstreams d, int M, int r, const int64_t* __restrict__ e, int64_t n,
               int64_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < (n + 1) / 2; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 2 * v;
    if (n0 + 1 < n) {
      const longlong2 q = __ldcs(reinterpret_cast<const longlong2*>(e + n0));
      uint64_t a = (uint64_t)q.x, b = (uint64_t)q.y;
      for (int m = 0; m < M; ++m) {
        if (m == r) continue;
        const longlong2 w = __ldcs(reinterpret_cast<const longlong2*>(d.s[m] + n0));
        a -= (uint64_t)w.x;
        b -= (uint64_t)w.y;
      }
      __stcs(reinterpret_cast<longlong2*>(out + n0), make_longlong2((int64_t)a, (int64_t)b));
    } else {
      uint64_t a = (uint64_t)e[n0];
      for (int m = 0; m < M; ++m)
        if (m != r) a -= (uint64_t)d.s[m][n0];
      out[n0] = (int64_t)a;
    }
  }
}

}  // namespace ne

using namespace ne;

extern "C" ne_status ne_abft_encode(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t* r_out,
                                    ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !r_out) return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (!c.s[m] || !aligned16(c.s[m])) return NE_EINVAL;
  k_abft_encode<<<grid_for((n_total + 3) / 4, kThreads), kThreads, 0, cs(stream)>>>(c, cfg->M, n_total, r_out, diag);
  return launch_status();
}

extern "C" ne_status ne_abft_encode_limbs(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int8_t* pdata,
                                          int32_t Ls, int8_t* psum, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || n_total % 16 != 0 || Ls < 1 || Ls > 4 || !pdata || !psum || !aligned16(pdata) ||
      !aligned16(psum))
    return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (!c.s[m] || !aligned16(c.s[m])) return NE_EINVAL;
  const int grid = grid_for(n_total / 4, kThreads);
  cudaStream_t s = cs(stream);
#define NE_AE(MV, LV) k_abft_encode_limbs<MV, LV><<<grid, kThreads, 0, s>>>(c, cfg->M, n_total, pdata, psum, diag)
#define NE_AE_L(MV)                 \
  switch (Ls) {                     \
    case 1: NE_AE(MV, 1); break;    \
    case 2: NE_AE(MV, 2); break;    \
    case 3: NE_AE(MV, 3); break;    \
    default: NE_AE(MV, 4); break;   \
  }
  switch (cfg->M) {
    case 3: NE_AE_L(3); break;
    case 4: NE_AE_L(4); break;
    case 8: NE_AE_L(8); break;
    default: NE_AE_L(0); break;
  }
#undef NE_AE_L
#undef NE_AE
  return launch_status();
}

extern "C" ne_status ne_to_limbs(ne_cstreams32 x, int32_t count, int64_t n_total, int32_t L, int8_t* planes,
                                 ne_diag* diag, ne_stream_t stream) {
  if (count < 1 || count > NE_MAX_M || n_total < 0 || n_total % 16 != 0 || L < 1 || L > 8 || !planes ||
      !aligned16(planes))
    return NE_EINVAL;
  for (int s = 0; s < count; ++s)
    if (!x.s[s] || !aligned16(x.s[s])) return NE_EINVAL;
  if (n_total == 0) return NE_OK;
  const int grid = grid_for(n_total / 4, kThreads);
  cudaStream_t s = cs(stream);
  switch (L) {
    case 1: k_to_limbs<1><<<grid, kThreads, 0, s>>>(x, count, n_total, planes, diag); break;
    case 2: k_to_limbs<2><<<grid, kThreads, 0, s>>>(x, count, n_total, planes, diag); break;
    case 3: k_to_limbs<3><<<grid, kThreads, 0, s>>>(x, count, n_total, planes, diag); break;
    case 4: k_to_limbs<4><<<grid, kThreads, 0, s>>>(x, count, n_total, planes, diag); break;
    default: k_to_limbs<8><<<grid, kThreads, 0, s>>>(x, count, n_total, planes, diag); break;
  }
  return launch_status();
}

extern "C" ne_status ne_abft_check(const ne_config* cfg, ne_cstreams d, const int64_t* e, int64_t n_total,
                                   uint32_t* bitmap, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !e || !aligned16(e)) return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (!d.s[m] || !aligned16(d.s[m])) return NE_EINVAL;
  k_abft_check<<<grid_for((n_total + 1) / 2, kThreads), kThreads, 0, cs(stream)>>>(d, cfg->M, e, n_total, bitmap,
                                                                                 diag);
  return launch_status();
}

extern "C" ne_status ne_abft_recover(const ne_config* cfg, ne_cstreams d, const int64_t* e, int64_t n_total,
                                     int32_t r, int64_t* d_r, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  for (int m = 0; m < cfg->M; ++m)
    if (m != r && !d.s[m]) return NE_EUNRECOVERABLE;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !e || !d_r || !aligned16(e) || !aligned16(d_r)) return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (m != r && !aligned16(d.s[m])) return NE_EINVAL;
  k_abft_recover<<<grid_for((n_total + 1) / 2, kThreads), kThreads, 0, cs(stream)>>>(d, cfg->M, r, e, n_total, d_r);
  return launch_status();
}
