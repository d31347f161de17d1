// k_stream.cu — streaming (HBM-bound) kernels of the hot path:
//   a1 entangle (SoA / AoS / int8 limb planes / one stream), a2 self-entangle,
//   a3 element-wise ops (scale, add), outer product, permutation gather,
//   and the device-side seeded input generator (gen/ne_gen.h).
// Layout and rooflines: DESIGN.md "Kernels".  Every kernel is a grid-stride
// loop over 128-bit vectors, grid = a multiple of the SM count.
#include <cuda_runtime.h>

#include <climits>

#include "../../gen/ne_gen.h"
#include "../../include/ne_gendev.h"
#include "ne_internal.cuh"

namespace ne {

// ---------------------------------------------------------------- a1 entangle
// eps_m[n] = c_m[n] + S_l{c_(m-1) mod M[n]}   (Eq. 15; Eq. 7 for M = 3).
// One thread handles 4 consecutive positions of ALL M streams, so every c_m is
// read exactly once (int4) and eps is written as 2 x 128-bit per stream.
// The a0 range assertion |c| <= hi is fused (warp-aggregated atomics).
// OUT selects the output layout: 0 = SoA int64, 1 = AoS int64 (generic M).
template <int MT, int OUT>
__global__ void __launch_bounds__(kThreads)
k_entangle(const __grid_constant__ ne_cstreams32 c, int M_rt, int l, int64_t hi, int64_t n,
           const __grid_constant__ ne_streams eps, int64_t* __restrict__ eps_aos, int8_t* __restrict__ planes,
           int L, ne_diag* __restrict__ diag, int set0 = 0) {
  const int M = MT > 0 ? MT : M_rt;
  const int so = (blockIdx.y + set0) * M;  // stream-set offset (ne_entangle_sets; 0 otherwise)
  int bad = 0;
  long long first = LLONG_MAX;
  const int64_t nvec = (n + 3) / 4;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = v * 4;
    const bool full = n0 + 4 <= n;
    int32_t first_c[4], prev[4];
    // c_{M-1} first: it is the "previous" stream of stream 0 (circulant Eq. 14)
    {
      const int32_t* p = c.s[so + M - 1] + n0;
      if (full) {
        int4 q = __ldcs(reinterpret_cast<const int4*>(p));
        first_c[0] = q.x; first_c[1] = q.y; first_c[2] = q.z; first_c[3] = q.w;
      } else {
        for (int i = 0; i < 4; ++i) first_c[i] = (n0 + i < n) ? p[i] : 0;
      }
      for (int i = 0; i < 4; ++i) prev[i] = first_c[i];
    }
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
      if (MT == 0 && m >= M) break;
      int32_t cur[4];
      if (m == M - 1) {
        for (int i = 0; i < 4; ++i) cur[i] = first_c[i];
      } else {
        const int32_t* p = c.s[so + m] + n0;
        if (full) {
          int4 q = __ldcs(reinterpret_cast<const int4*>(p));
          cur[0] = q.x; cur[1] = q.y; cur[2] = q.z; cur[3] = q.w;
        } else {
          for (int i = 0; i < 4; ++i) cur[i] = (n0 + i < n) ? p[i] : 0;
        }
      }
      int64_t e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        e[i] = (int64_t)cur[i] + (int64_t)((uint64_t)(int64_t)prev[i] << l);
        const int64_t ci = cur[i];
        if ((ci > hi || ci < -hi) && n0 + i < n) {
          ++bad;
          long long idx = (long long)(so + m) * n + n0 + i;
          first = idx < first ? idx : first;
        }
      }
      if (OUT == 0) {
        int64_t* q = eps.s[so + m] + n0;
        if (full) {
          __stcs(reinterpret_cast<longlong2*>(q), make_longlong2(e[0], e[1]));
          __stcs(reinterpret_cast<longlong2*>(q) + 1, make_longlong2(e[2], e[3]));
        } else {
          for (int i = 0; i < 4; ++i)
            if (n0 + i < n) q[i] = e[i];
        }
      } else if (OUT == 1) {
        for (int i = 0; i < 4; ++i)
          if (n0 + i < n) eps_aos[(n0 + i) * M + m] = e[i];
      }
      for (int i = 0; i < 4; ++i) prev[i] = cur[i];
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// AoS for M = 4: a warp owns 128 consecutive positions per iteration, lane t
// positions base + 32 i + t (i < 4): every 32-bit load instruction is one
// coalesced 128-byte line per stream, and every position is written with ONE
// 256-bit store (its whole 32-byte DRAM sector; 1 KB contiguous per warp
// instruction) — the layout the C4 gather reads.
__global__ void __launch_bounds__(kThreads)
k_entangle_aos4(const __grid_constant__ ne_cstreams32 c, int l, int64_t hi, int64_t n,
                int64_t* __restrict__ eps_aos, ne_diag* __restrict__ diag) {
  int bad = 0;
  long long first = LLONG_MAX;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * 128; base < n; base += nwarps * 128) {
    int32_t cv[4][4];  // [stream][i]
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t p = base + 32 * i + lane;
        cv[m][i] = p < n ? __ldcs(c.s[m] + p) : 0;
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t p = base + 32 * i + lane;
      if (p >= n) continue;
      uint64_t e[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int64_t x = cv[m][i];
        if (x > hi || x < -hi) {
          ++bad;
          const long long idx = (long long)m * n + p;
          first = idx < first ? idx : first;
        }
        e[m] = (uint64_t)x + ((uint64_t)(int64_t)cv[(m + 3) & 3][i] << l);
      }
      asm volatile("st.global.cs.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(eps_aos + p * 4), "l"(e[0]), "l"(e[1]),
                   "l"(e[2]), "l"(e[3])
                   : "memory");
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// Entangle straight into the L int8 digit planes of the tensor-core GEMM.
// Balanced base-2^8 digits in one add: with bias = sum_{i<L} 128 * 256^i,
// x = sum_i d_i 256^i, d_i in [-128,127]  <=>  y = x + bias in [0, 256^L) and
// byte i of y = d_i + 128, so d_i = byte_i(y) ^ 0x80 (two's complement).
// A thread owns 4 consecutive positions (one 128-bit load per stream, all M
// loads issued before any store); plane j receives the 4 bytes j of the four
// y values (PRMT), a 32-bit store per plane (128 contiguous bytes per warp).
template <int MT, int L>
__global__ void __launch_bounds__(kThreads)
k_entangle_limbs(const __grid_constant__ ne_cstreams32 c, int M_rt, int l, int64_t hi, int64_t n,
                 int8_t* __restrict__ planes, ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  constexpr uint64_t bias = 0x8080808080808080ull >> (64 - 8 * L);
  constexpr uint64_t span = L == 8 ? 0 : (1ull << (8 * L));  // 256^L
  int bad = 0;
  long long first = LLONG_MAX;
  const int64_t nvec = n / 4;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    int4 q[MA];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) q[m] = __ldcs(reinterpret_cast<const int4*>(c.s[m] + n0));
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      const int4 cur = q[m], prv = q[m == 0 ? M - 1 : m - 1];
      const int32_t cc[4] = {cur.x, cur.y, cur.z, cur.w}, pp[4] = {prv.x, prv.y, prv.z, prv.w};
      uint64_t y[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t ci = cc[i];
        const uint64_t x = (uint64_t)ci + ((uint64_t)(int64_t)pp[i] << l);
        y[i] = x + bias;
        const bool out_of_limbs = L < 8 && y[i] >= span;
        if (ci > hi || ci < -hi || out_of_limbs) {
          ++bad;
          const long long idx = (long long)m * n + n0 + i;
          first = idx < first ? idx : first;
        }
      }
      const uint32_t lo01 = __byte_perm((uint32_t)y[0], (uint32_t)y[1], 0x5140);  // b0(y0) b0(y1) b1(y0) b1(y1)
      const uint32_t lo23 = __byte_perm((uint32_t)y[2], (uint32_t)y[3], 0x5140);
      const uint32_t hi01 = __byte_perm((uint32_t)y[0], (uint32_t)y[1], 0x7362);  // b2(y0) b2(y1) b3(y0) b3(y1)
      const uint32_t hi23 = __byte_perm((uint32_t)y[2], (uint32_t)y[3], 0x7362);
      uint32_t w[8];
      w[0] = __byte_perm(lo01, lo23, 0x5410);  // byte 0 of y0..y3
      w[1] = __byte_perm(lo01, lo23, 0x7632);  // byte 1
      w[2] = __byte_perm(hi01, hi23, 0x5410);  // byte 2
      w[3] = __byte_perm(hi01, hi23, 0x7632);  // byte 3
      if (L > 4) {
        const uint32_t a01 = __byte_perm((uint32_t)(y[0] >> 32), (uint32_t)(y[1] >> 32), 0x5140);
        const uint32_t a23 = __byte_perm((uint32_t)(y[2] >> 32), (uint32_t)(y[3] >> 32), 0x5140);
        const uint32_t b01 = __byte_perm((uint32_t)(y[0] >> 32), (uint32_t)(y[1] >> 32), 0x7362);
        const uint32_t b23 = __byte_perm((uint32_t)(y[2] >> 32), (uint32_t)(y[3] >> 32), 0x7362);
        w[4] = __byte_perm(a01, a23, 0x5410);
        w[5] = __byte_perm(a01, a23, 0x7632);
        w[6] = __byte_perm(b01, b23, 0x5410);
        w[7] = __byte_perm(b01, b23, 0x7632);
      }
#pragma unroll
      for (int j = 0; j < L; ++j)
        __stcs(reinterpret_cast<unsigned int*>(planes + ((int64_t)m * L + j) * n + n0), w[j] ^ 0x80808080u);
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// The two-digit base-2^l plan in pure 32-bit arithmetic:
// eps = c + 2^b p (b = l <= 31) has digits d0 = sext_b(c) and
// d1 = p + (c - d0) / 2^b = p + (c >> b) + bit_{b-1}(c); it is exact iff both
// fit int8.  8 positions per thread: one 256-bit load per stream (two 128-bit
// loads when a stream is only 16-B aligned), one 64-bit store per digit plane.
// Wrapping of d1 in int32 cannot fake a valid digit: a wrapped value is near
// -2^31.  Range failures (|c| > hi, digit out of int8) take a slow path.
// (r02 A/B, C3's 3 x 4096^2 operand, L2 flushed: 55.3 us = 5.46 TB/s; 16
// positions per thread with 128-bit plane stores 57.3 us — fewer resident
// threads for the same bytes in flight.)  The plane stores stay evict-first:
// ordinary stores of the planes and of prep_b's Bt, so the GEMM would find
// part of them in L2, took the C3 step from 0.5614 to 0.566-0.575 ms (three
// alternating default lines, r02z55: GEMM 0.283-0.289 vs 0.287-0.295 ms, the
// entangle 0.061 vs 0.058 ms).
__device__ __forceinline__ uint32_t pack4(int32_t a, int32_t b, int32_t c, int32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

#ifndef NE_EP_MINB  // r02 A/B (scripts/r02/z42.sh, L2 flushed): 1 (64 regs) 57.3 us, 5 (48, spills) 61.4, 6 (40) 67.6
#define NE_EP_MINB 1
#endif
template <int MT, bool V256>
__global__ void __launch_bounds__(kThreads, NE_EP_MINB)
k_entangle_pair(const __grid_constant__ ne_cstreams32 c, int M_rt, int b, int64_t hi, int64_t n,
                int8_t* __restrict__ planes, ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const bool rc = hi < 2147483647ll;  // |c| <= hi can fail for an int32 only then
  const int32_t h32 = rc ? (int32_t)hi : 0;
  const int sh = 32 - b;
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n / 8; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 8 * v;
    int32_t q[MA][8];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      const int32_t* p = c.s[m] + n0;
      if (V256) {
        uint64_t u0, u1, u2, u3;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(u0), "=l"(u1), "=l"(u2), "=l"(u3)
                     : "l"(p));
        const uint64_t u[4] = {u0, u1, u2, u3};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          q[m][2 * k] = (int32_t)(uint32_t)u[k];
          q[m][2 * k + 1] = (int32_t)(uint32_t)(u[k] >> 32);
        }
      } else {
        const int4 a = __ldcs(reinterpret_cast<const int4*>(p));
        const int4 e = __ldcs(reinterpret_cast<const int4*>(p + 4));
        q[m][0] = a.x; q[m][1] = a.y; q[m][2] = a.z; q[m][3] = a.w;
        q[m][4] = e.x; q[m][5] = e.y; q[m][6] = e.z; q[m][7] = e.w;
      }
    }
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      const int mp = m == 0 ? M - 1 : m - 1;
      int32_t d0[8], d1[8];
      uint32_t badm = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int32_t cc = q[m][i];
        d0[i] = (int32_t)((uint32_t)cc << sh) >> sh;
        d1[i] = q[mp][i] + (cc >> b) + ((cc >> (b - 1)) & 1);
        uint32_t f = ((uint32_t)(d0[i] + 128) | (uint32_t)(d1[i] + 128)) > 255u;
        if (rc) f |= (cc > h32) | (cc < -h32);
        badm |= f << i;
      }
      if (badm) {
        bad += __popc(badm);
        const long long idx = (long long)m * n + n0 + (__ffs(badm) - 1);
        first = idx < first ? idx : first;
      }
      int8_t* p0 = planes + ((int64_t)m * 2) * n + n0;
      __stcs(reinterpret_cast<uint2*>(p0), make_uint2(pack4(d0[0], d0[1], d0[2], d0[3]), pack4(d0[4], d0[5], d0[6], d0[7])));
      __stcs(reinterpret_cast<uint2*>(p0 + n), make_uint2(pack4(d1[0], d1[1], d1[2], d1[3]), pack4(d1[4], d1[5], d1[6], d1[7])));
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// Entangle into L digit planes of a general base 2^b (b != 8), 4 positions per
// thread, all M streams loaded first; digits via digits_b.
template <int MT, int L>
__global__ void __launch_bounds__(kThreads)
k_entangle_digits(const __grid_constant__ ne_cstreams32 c, int M_rt, int l, int64_t hi, int64_t n, int b,
                  int8_t* __restrict__ planes, ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n / 4; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    int4 q[MA];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) q[m] = __ldcs(reinterpret_cast<const int4*>(c.s[m] + n0));
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      const int4 cur = q[m], prv = q[m == 0 ? M - 1 : m - 1];
      const int32_t cc[4] = {cur.x, cur.y, cur.z, cur.w}, pp[4] = {prv.x, prv.y, prv.z, prv.w};
      uint32_t w[L];
#pragma unroll
      for (int j = 0; j < L; ++j) w[j] = 0;
      if (L == 2 && b == l && b <= 31) {
        // the base-2^l plan in 32-bit arithmetic: x = c + 2^b p has
        // d0 = sext_b(c) (its low b bits are c's), d1 = p + (c - d0) / 2^b
        const int sh = 32 - b;
        int32_t d0[4], d1[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          d0[i] = (int32_t)((uint32_t)cc[i] << sh) >> sh;
          const int64_t d1w = (int64_t)pp[i] + (((int64_t)cc[i] - d0[i]) >> b);
          d1[i] = (int32_t)d1w;
          const bool ok = (uint32_t)(d0[i] + 128) < 256u && (uint64_t)(d1w + 128) < 256u;
          if (cc[i] > hi || cc[i] < -hi || !ok) {
            ++bad;
            const long long idx = (long long)m * n + n0 + i;
            first = idx < first ? idx : first;
          }
        }
        w[0] = __byte_perm(__byte_perm(d0[0], d0[1], 0x0040), __byte_perm(d0[2], d0[3], 0x0040), 0x5410);
        w[L - 1] = __byte_perm(__byte_perm(d1[0], d1[1], 0x0040), __byte_perm(d1[2], d1[3], 0x0040), 0x5410);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t ci = cc[i];
          const int64_t x = (int64_t)((uint64_t)ci + ((uint64_t)(int64_t)pp[i] << l));
          int8_t d[L];
          const bool ok = digits_b(x, b, L, d);
          if (ci > hi || ci < -hi || !ok) {
            ++bad;
            const long long idx = (long long)m * n + n0 + i;
            first = idx < first ? idx : first;
          }
#pragma unroll
          for (int j = 0; j < L; ++j) w[j] |= (uint32_t)(uint8_t)d[j] << (8 * i);
        }
      }
#pragma unroll
      for (int j = 0; j < L; ++j)
        __stcs(reinterpret_cast<unsigned int*>(planes + ((int64_t)m * L + j) * n + n0), w[j]);
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// one stream into L digit planes (same digit trick as k_entangle_limbs)
template <int L>
__global__ void __launch_bounds__(kThreads)
k_entangle_limbs_stream(const int32_t* __restrict__ cm, const int32_t* __restrict__ cp, int m, int l, int64_t hi,
                        int64_t n, int b, int8_t* __restrict__ planes, ne_diag* __restrict__ diag) {
  constexpr uint64_t bias = 0x8080808080808080ull >> (64 - 8 * L);
  constexpr uint64_t span = L == 8 ? 0 : (1ull << (8 * L));
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n / 4; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    const int4 a = __ldcs(reinterpret_cast<const int4*>(cm + n0)), bq = __ldcs(reinterpret_cast<const int4*>(cp + n0));
    const int32_t cc[4] = {a.x, a.y, a.z, a.w}, pp[4] = {bq.x, bq.y, bq.z, bq.w};
    uint32_t w[L];
#pragma unroll
    for (int j = 0; j < L; ++j) w[j] = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t ci = cc[i];
      const uint64_t x = (uint64_t)ci + ((uint64_t)(int64_t)pp[i] << l);
      bool ok;
      if (b == 8) {
        const uint64_t y = x + bias;
        ok = !(L < 8 && y >= span);
#pragma unroll
        for (int j = 0; j < L; ++j) w[j] |= (uint32_t)(((y >> (8 * j)) & 0xff) ^ 0x80) << (8 * i);
      } else {
        int8_t d[L];
        ok = digits_b((int64_t)x, b, L, d);
#pragma unroll
        for (int j = 0; j < L; ++j) w[j] |= (uint32_t)(uint8_t)d[j] << (8 * i);
      }
      if (ci > hi || ci < -hi || !ok) {
        ++bad;
        const long long idx = (long long)m * n + n0 + i;
        first = idx < first ? idx : first;
      }
    }
#pragma unroll
    for (int j = 0; j < L; ++j) __stcs(reinterpret_cast<unsigned int*>(planes + (int64_t)j * n + n0), w[j]);
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// one stream: eps_m = c_m + S_l{c_prev}
__global__ void __launch_bounds__(kThreads)
k_entangle_stream(const int32_t* __restrict__ cm, const int32_t* __restrict__ cp, int m, int l,
                  int64_t hi, int64_t n, int64_t* __restrict__ eps, ne_diag* __restrict__ diag) {
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = __ldcs(cm + i), b = __ldcs(cp + i);
    if (a > hi || a < -hi) {
      ++bad;
      long long idx = (long long)m * n + i;
      first = idx < first ? idx : first;
    }
    __stcs(eps + i, a + (int64_t)((uint64_t)b << l));
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// a2: g_ent = S_l{g} + g (footnote P:507-511)
__global__ void k_entangle_shared(const int32_t* __restrict__ g, int l, int64_t n,
                                  int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = g[i];
    out[i] = (int64_t)((uint64_t)v << l) + v;
  }
}

// ---------------------------------------------------------------- a3 element-wise
// x_m[n] *= (g ? g[n] : s) — 2 positions (128 bits) per thread per stream
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_scale(const __grid_constant__ ne_streams x, int M_rt, int64_t n, int64_t s,
        const int32_t* __restrict__ g) {
  const int M = MT > 0 ? MT : M_rt;
  const int64_t npair = (n + 1) / 2;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < npair;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 2 * v;
    int64_t f0 = s, f1 = s;
    if (g) {
      f0 = g[n0];
      f1 = (n0 + 1 < n) ? g[n0 + 1] : 0;
    }
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
      if (MT == 0 && m >= M) break;
      int64_t* p = x.s[m] + n0;
      if (n0 + 1 < n) {
        longlong2 q = __ldcs(reinterpret_cast<const longlong2*>(p));
        q.x = (int64_t)((uint64_t)q.x * (uint64_t)f0);
        q.y = (int64_t)((uint64_t)q.y * (uint64_t)f1);
        __stcs(reinterpret_cast<longlong2*>(p), q);
      } else {
        p[0] = (int64_t)((uint64_t)p[0] * (uint64_t)f0);
      }
    }
  }
}

// x_m[n] += sign * a_m[n]
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_add(const __grid_constant__ ne_streams x, const __grid_constant__ ne_cstreams a, int M_rt,
      int64_t n, int sign) {
  const int M = MT > 0 ? MT : M_rt;
  const int64_t npair = (n + 1) / 2;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < npair;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 2 * v;
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
      if (MT == 0 && m >= M) break;
      int64_t* p = x.s[m] + n0;
      const int64_t* q = a.s[m] + n0;
      if (n0 + 1 < n) {
        longlong2 u = __ldcs(reinterpret_cast<const longlong2*>(p));
        longlong2 w = __ldcs(reinterpret_cast<const longlong2*>(q));
        u.x = sign > 0 ? (int64_t)((uint64_t)u.x + (uint64_t)w.x) : (int64_t)((uint64_t)u.x - (uint64_t)w.x);
        u.y = sign > 0 ? (int64_t)((uint64_t)u.y + (uint64_t)w.y) : (int64_t)((uint64_t)u.y - (uint64_t)w.y);
        __stcs(reinterpret_cast<longlong2*>(p), u);
      } else {
        p[0] = sign > 0 ? (int64_t)((uint64_t)p[0] + (uint64_t)q[0]) : (int64_t)((uint64_t)p[0] - (uint64_t)q[0]);
      }
    }
  }
}

// x_m[n] = x_m[n] * (g ? g[n] : s) + sign * a_m[n]: a scale and an add of the
// LSB chain in one pass (40 -> 24 B per position and stream)
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_scale_add(const __grid_constant__ ne_streams x, const __grid_constant__ ne_cstreams a, int M_rt, int64_t n,
            int64_t s, const int32_t* __restrict__ g, int sign) {
  const int M = MT > 0 ? MT : M_rt;
  const int64_t npair = (n + 1) / 2;
  const uint64_t sg = (uint64_t)(int64_t)sign;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < npair;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 2 * v;
    uint64_t f0 = (uint64_t)s, f1 = (uint64_t)s;
    if (g) {
      f0 = (uint64_t)(int64_t)g[n0];
      f1 = (n0 + 1 < n) ? (uint64_t)(int64_t)g[n0 + 1] : 0;
    }
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
      if (MT == 0 && m >= M) break;
      int64_t* p = x.s[m] + n0;
      const int64_t* q = a.s[m] + n0;
      if (n0 + 1 < n) {
        longlong2 u = __ldcs(reinterpret_cast<const longlong2*>(p));
        const longlong2 w = __ldcs(reinterpret_cast<const longlong2*>(q));
        u.x = (int64_t)((uint64_t)u.x * f0 + sg * (uint64_t)w.x);
        u.y = (int64_t)((uint64_t)u.y * f1 + sg * (uint64_t)w.y);
        __stcs(reinterpret_cast<longlong2*>(p), u);
      } else {
        p[0] = (int64_t)((uint64_t)p[0] * f0 + sg * (uint64_t)q[0]);
      }
    }
  }
}

// outer product: out_m[i*n2 + j] = x_m[i] * h[j]; write-bound, 2 outputs / thread
__global__ void __launch_bounds__(kThreads)
k_outer(const __grid_constant__ ne_cstreams x, const __grid_constant__ ne_streams out, int M,
        int64_t n1, const int32_t* __restrict__ h, int64_t n2) {
  const int64_t total = n1 * n2;
  const int64_t npair = (total + 1) / 2;
  const bool even = (n2 % 2) == 0;
  for (int m = 0; m < M; ++m) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < npair;
         v += (int64_t)gridDim.x * blockDim.x) {
      const int64_t o = 2 * v;
      if (even) {
        const int64_t i = o / n2, j = o - i * n2;
        const uint64_t xi = (uint64_t)x.s[m][i];
        __stcs(reinterpret_cast<longlong2*>(out.s[m] + o),
               make_longlong2((int64_t)(xi * (uint64_t)(int64_t)h[j]), (int64_t)(xi * (uint64_t)(int64_t)h[j + 1])));
      } else {
        for (int64_t q = o; q < o + 2 && q < total; ++q) {
          const int64_t i = q / n2, j = q - i * n2;
          out.s[m][q] = (int64_t)((uint64_t)x.s[m][i] * (uint64_t)(int64_t)h[j]);
        }
      }
    }
  }
}

// permutation gather out_m[i] = x_m[perm[i]] (SoA)
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_permute(const __grid_constant__ ne_cstreams x, const __grid_constant__ ne_streams out,
          int M_rt, const int32_t* __restrict__ perm, int64_t n) {
  const int M = MT > 0 ? MT : M_rt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = __ldcs(perm + i);
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
      if (MT == 0 && m >= M) break;
      __stcs(out.s[m] + i, __ldg(x.s[m] + src));
    }
  }
}

// ---------------------------------------------------------------- generator
__global__ void k_gen_uniform(uint64_t key, int64_t lo, int64_t hi, int64_t offset, int64_t count,
                              int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)ne_gen_uniform(key, (uint64_t)(offset + i), lo, hi);
}

__global__ void k_gen_perm(uint64_t key, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)ne_gen_perm(key, (uint64_t)n, (uint64_t)i);
}

}  // namespace ne

using namespace ne;

#define NE_DISPATCH_M(M, KERNEL, GRID, STREAM, ...)                  \
  switch (M) {                                                     \
    case 3: KERNEL<3><<<GRID, kThreads, 0, STREAM>>>(__VA_ARGS__); break;  \
    case 4: KERNEL<4><<<GRID, kThreads, 0, STREAM>>>(__VA_ARGS__); break;  \
    case 8: KERNEL<8><<<GRID, kThreads, 0, STREAM>>>(__VA_ARGS__); break;  \
    default: KERNEL<0><<<GRID, kThreads, 0, STREAM>>>(__VA_ARGS__); break; \
  }

static bool streams_ok32(const ne_cstreams32& c, int M) {
  for (int m = 0; m < M; ++m)
    if (!c.s[m] || !aligned16(c.s[m])) return false;
  return true;
}
template <typename S>
static bool streams_ok(const S& c, int M) {
  for (int m = 0; m < M; ++m)
    if (!c.s[m] || !aligned16(c.s[m])) return false;
  return true;
}

template <int OUT>
static ne_status launch_entangle(const ne_config* cfg, ne_cstreams32 c, int64_t n, ne_streams eps,
                                 int64_t* aos, int8_t* planes, int L, ne_diag* diag,
                                 ne_stream_t stream) {
  const int64_t hi = range_hi(cfg);
  const int grid = grid_for((n + 3) / 4, kThreads);
  cudaStream_t s = cs(stream);
  switch (cfg->M) {
    case 3: k_entangle<3, OUT><<<grid, kThreads, 0, s>>>(c, 3, cfg->l, hi, n, eps, aos, planes, L, diag); break;
    case 4: k_entangle<4, OUT><<<grid, kThreads, 0, s>>>(c, 4, cfg->l, hi, n, eps, aos, planes, L, diag); break;
    case 8: k_entangle<8, OUT><<<grid, kThreads, 0, s>>>(c, 8, cfg->l, hi, n, eps, aos, planes, L, diag); break;
    default: k_entangle<0, OUT><<<grid, kThreads, 0, s>>>(c, cfg->M, cfg->l, hi, n, eps, aos, planes, L, diag); break;
  }
  return launch_status();
}

extern "C" ne_status ne_entangle(const ne_config* cfg, ne_cstreams32 c, int64_t n_total,
                                 ne_streams eps, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !streams_ok32(c, cfg->M) || !streams_ok(eps, cfg->M)) return NE_EINVAL;
  return launch_entangle<0>(cfg, c, n_total, eps, nullptr, nullptr, 0, diag, stream);
}

extern "C" ne_status ne_entangle_sets(const ne_config* cfg, ne_cstreams32 c, int32_t sets, int64_t n_total,
                                      ne_streams eps, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (sets < 1 || sets * cfg->M > NE_MAX_M) return NE_EINVAL;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !streams_ok32(c, sets * cfg->M) || !streams_ok(eps, sets * cfg->M)) return NE_EINVAL;
  const int64_t hi = range_hi(cfg);
  cudaStream_t s = cs(stream);
  // small streams: all sets in one launch (grid.y = set; launch latency
  // dominates); large streams: one launch per set (measured faster at 2^27)
  const bool one = n_total <= (1 << 22);
  const int ny = one ? sets : 1;
  const dim3 grid((unsigned)grid_for((n_total + 3) / 4, kThreads, one ? (8 + sets - 1) / sets : 8), (unsigned)ny);
  for (int s0 = 0; s0 < sets; s0 += ny) {
    switch (cfg->M) {
      case 3: k_entangle<3, 0><<<grid, kThreads, 0, s>>>(c, 3, cfg->l, hi, n_total, eps, nullptr, nullptr, 0, diag, s0); break;
      case 4: k_entangle<4, 0><<<grid, kThreads, 0, s>>>(c, 4, cfg->l, hi, n_total, eps, nullptr, nullptr, 0, diag, s0); break;
      case 8: k_entangle<8, 0><<<grid, kThreads, 0, s>>>(c, 8, cfg->l, hi, n_total, eps, nullptr, nullptr, 0, diag, s0); break;
      default: k_entangle<0, 0><<<grid, kThreads, 0, s>>>(c, cfg->M, cfg->l, hi, n_total, eps, nullptr, nullptr, 0, diag, s0); break;
    }
  }
  return launch_status();
}

extern "C" ne_status ne_entangle_aos(const ne_config* cfg, ne_cstreams32 c, int64_t n_total,
                                     int64_t* eps_aos, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !streams_ok32(c, cfg->M) || !eps_aos || !aligned16(eps_aos)) return NE_EINVAL;
  if (cfg->M == 4) {
    k_entangle_aos4<<<grid_for((n_total + 3) / 4, kThreads), kThreads, 0, cs(stream)>>>(c, cfg->l, range_hi(cfg), n_total,
                                                                            eps_aos, diag);
    return launch_status();
  }
  ne_streams none{};
  return launch_entangle<1>(cfg, c, n_total, none, eps_aos, nullptr, 0, diag, stream);
}

extern "C" ne_status ne_entangle_limbs(const ne_config* cfg, ne_cstreams32 c, int64_t n_total,
                                       int32_t L, int32_t limb_bits, int8_t* planes, ne_diag* diag,
                                       ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || n_total % 16 != 0 || L < 1 || L > 8 || limb_bits < 8 || limb_bits > 63 ||
      !streams_ok32(c, cfg->M) || !planes || !aligned16(planes))
    return NE_EINVAL;
  if (limb_bits != 8) {
    if (L > 4) return NE_EINVAL;  // base-2^b digit planes: L <= 4
    cudaStream_t s = cs(stream);
    const int64_t hi = range_hi(cfg);
    if (L == 2 && limb_bits == cfg->l && limb_bits <= 31) {
      bool a32 = true;
      for (int m = 0; m < cfg->M; ++m) a32 &= (reinterpret_cast<uintptr_t>(c.s[m]) & 31u) == 0;
      const int g8 = grid_for(n_total / 8, kThreads);
#define NE_PAIR(MV)                                                                                   \
  if (a32)                                                                                            \
    k_entangle_pair<MV, true><<<g8, kThreads, 0, s>>>(c, cfg->M, limb_bits, hi, n_total, planes, diag); \
  else                                                                                                \
    k_entangle_pair<MV, false><<<g8, kThreads, 0, s>>>(c, cfg->M, limb_bits, hi, n_total, planes, diag)
      switch (cfg->M) {
        case 3: NE_PAIR(3); break;
        case 4: NE_PAIR(4); break;
        case 8: NE_PAIR(8); break;
        default: NE_PAIR(0); break;
      }
#undef NE_PAIR
      return launch_status();
    }
    const int grid = grid_for(n_total / 4, kThreads);
#define NE_DIG(MV, LV) k_entangle_digits<MV, LV><<<grid, kThreads, 0, s>>>(c, cfg->M, cfg->l, hi, n_total, limb_bits, planes, diag)
#define NE_DIG_L(MV)                                                                   \
  switch (L) {                                                                         \
    case 1: NE_DIG(MV, 1); break;                                                      \
    case 2: NE_DIG(MV, 2); break;                                                      \
    case 3: NE_DIG(MV, 3); break;                                                      \
    case 4: NE_DIG(MV, 4); break;                                                      \
    default: NE_DIG(MV, 4); break;                                                     \
  }
    switch (cfg->M) {
      case 3: NE_DIG_L(3); break;
      case 4: NE_DIG_L(4); break;
      case 8: NE_DIG_L(8); break;
      default: NE_DIG_L(0); break;
    }
#undef NE_DIG_L
#undef NE_DIG
    return launch_status();
  }
  const int64_t hi = range_hi(cfg);
  const int grid = grid_for(n_total / 4, kThreads);
  cudaStream_t s = cs(stream);
#define NE_LIMB_CASE(MV, LV) k_entangle_limbs<MV, LV><<<grid, kThreads, 0, s>>>(c, cfg->M, cfg->l, hi, n_total, planes, diag)
#define NE_LIMB_L(MV)              \
  switch (L) {                     \
    case 1: NE_LIMB_CASE(MV, 1); break; \
    case 2: NE_LIMB_CASE(MV, 2); break; \
    case 3: NE_LIMB_CASE(MV, 3); break; \
    case 4: NE_LIMB_CASE(MV, 4); break; \
    case 5: NE_LIMB_CASE(MV, 5); break; \
    case 6: NE_LIMB_CASE(MV, 6); break; \
    case 7: NE_LIMB_CASE(MV, 7); break; \
    default: NE_LIMB_CASE(MV, 8); break; \
  }
  switch (cfg->M) {
    case 3: NE_LIMB_L(3); break;
    case 4: NE_LIMB_L(4); break;
    case 8: NE_LIMB_L(8); break;
    default: NE_LIMB_L(0); break;
  }
#undef NE_LIMB_L
#undef NE_LIMB_CASE
  return launch_status();
}

extern "C" ne_status ne_entangle_stream(const ne_config* cfg, int32_t m, const int32_t* c_m,
                                        const int32_t* c_prev, int64_t* eps_m, int64_t n_total,
                                        ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (m < 0 || m >= cfg->M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !c_m || !c_prev || !eps_m || !aligned16(c_m) || !aligned16(c_prev) || !aligned16(eps_m))
    return NE_EINVAL;
  k_entangle_stream<<<grid_for(n_total, kThreads), kThreads, 0, cs(stream)>>>(c_m, c_prev, m, cfg->l,
                                                                            range_hi(cfg), n_total, eps_m, diag);
  return launch_status();
}

extern "C" ne_status ne_entangle_limbs_stream(const ne_config* cfg, int32_t m, const int32_t* c_m,
                                              const int32_t* c_prev, int64_t n_total, int32_t L, int32_t limb_bits,
                                              int8_t* planes_m, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (m < 0 || m >= cfg->M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || n_total % 16 != 0 || L < 1 || L > 8 || limb_bits < 8 || limb_bits > 63 || !c_m || !c_prev ||
      !planes_m || !aligned16(c_m) || !aligned16(c_prev) || !aligned16(planes_m))
    return NE_EINVAL;
  const int grid = grid_for(n_total / 4, kThreads);
  const int64_t hi = range_hi(cfg);
  cudaStream_t s = cs(stream);
  switch (L) {
    case 1: k_entangle_limbs_stream<1><<<grid, kThreads, 0, s>>>(c_m, c_prev, m, cfg->l, hi, n_total, limb_bits, planes_m, diag); break;
    case 2: k_entangle_limbs_stream<2><<<grid, kThreads, 0, s>>>(c_m, c_prev, m, cfg->l, hi, n_total, limb_bits, planes_m, diag); break;
    case 3: k_entangle_limbs_stream<3><<<grid, kThreads, 0, s>>>(c_m, c_prev, m, cfg->l, hi, n_total, limb_bits, planes_m, diag); break;
    case 4: k_entangle_limbs_stream<4><<<grid, kThreads, 0, s>>>(c_m, c_prev, m, cfg->l, hi, n_total, limb_bits, planes_m, diag); break;
    default: k_entangle_limbs_stream<8><<<grid, kThreads, 0, s>>>(c_m, c_prev, m, cfg->l, hi, n_total, limb_bits, planes_m, diag); break;
  }
  return launch_status();
}

// The split ("mixed-radix") digit plan of the GEMM operand:
// eps_m = c_m + 2^l c_{m-1} held as 2D int8 planes — the D balanced base-256
// digits of c_m (bit weights 0, 8, ..) and the D digits of c_{m-1} (weights
// l, l + 8, ..): planes[(m*2D + i)*n + idx].  Stream m's planes hold only
// stream m's operand (stream-local: a fault in stream m's product still
// corrupts delta_m alone, Props 2/4).  4 positions per thread; a value the D
// digits cannot hold, or |c| > hi, is a range violation naming m*n + idx.
template <int MT, int D>
__global__ void __launch_bounds__(kThreads)
k_entangle_split(const __grid_constant__ ne_cstreams32 c, int M_rt, int64_t hi, int64_t n,
                 int8_t* __restrict__ planes, ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  constexpr int64_t bias = (int64_t)(0x8080808080808080ull >> (64 - 8 * D));
  constexpr int64_t span = (int64_t)1 << (8 * D);
  int bad = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n / 4; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    int4 q[MA];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) q[m] = __ldcs(reinterpret_cast<const int4*>(c.s[m] + n0));
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      const int4 cur = q[m], prv = q[m == 0 ? M - 1 : m - 1];
      const int32_t cc[4] = {cur.x, cur.y, cur.z, cur.w}, pp[4] = {prv.x, prv.y, prv.z, prv.w};
      uint32_t w[2 * D];
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) w[j] = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t ylo = (int64_t)cc[i] + bias, yhi = (int64_t)pp[i] + bias;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          w[j] |= (uint32_t)(((ylo >> (8 * j)) & 0xff) ^ 0x80) << (8 * i);
          w[D + j] |= (uint32_t)(((yhi >> (8 * j)) & 0xff) ^ 0x80) << (8 * i);
        }
        // c_m's digits are checked here; c_{m-1}'s by stream m-1 (the same value)
        if (cc[i] > hi || cc[i] < -hi || ylo < 0 || ylo >= span) {
          ++bad;
          const long long idx = (long long)m * n + n0 + i;
          first = idx < first ? idx : first;
        }
      }
#pragma unroll
      for (int j = 0; j < 2 * D; ++j)
        __stcs(reinterpret_cast<unsigned int*>(planes + ((int64_t)m * 2 * D + j) * n + n0), w[j]);
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

extern "C" ne_status ne_entangle_plan(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, const ne_gemm_plan* plan,
                                      int8_t* planes, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!plan) return NE_EINVAL;
  if (plan->kind == NE_PLAN_EPS) return ne_entangle_limbs(cfg, c, n_total, plan->LA, plan->digit_bits, planes, diag, stream);
  if (plan->kind != NE_PLAN_SPLIT || plan->LA < 2 || plan->LA > 8 || plan->LA % 2) return NE_EINVAL;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || n_total % 16 != 0 || !streams_ok32(c, cfg->M) || !planes || !aligned16(planes)) return NE_EINVAL;
  const int64_t hi = range_hi(cfg);
  const int grid = grid_for(n_total / 4, kThreads);
  cudaStream_t s = cs(stream);
#define NE_SPLIT(MV, DV) k_entangle_split<MV, DV><<<grid, kThreads, 0, s>>>(c, cfg->M, hi, n_total, planes, diag)
#define NE_SPLIT_D(MV)            \
  switch (plan->LA / 2) {          \
    case 1: NE_SPLIT(MV, 1); break; \
    case 2: NE_SPLIT(MV, 2); break; \
    case 3: NE_SPLIT(MV, 3); break; \
    default: NE_SPLIT(MV, 4); break; \
  }
  switch (cfg->M) {
    case 3: NE_SPLIT_D(3); break;
    case 4: NE_SPLIT_D(4); break;
    case 8: NE_SPLIT_D(8); break;
    default: NE_SPLIT_D(0); break;
  }
#undef NE_SPLIT_D
#undef NE_SPLIT
  return launch_status();
}

extern "C" ne_status ne_entangle_shared(const ne_config* cfg, const int32_t* g, int64_t* g_ent,
                                        int64_t n_total, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !g || !g_ent) return NE_EINVAL;
  k_entangle_shared<<<grid_for(n_total, kThreads), kThreads, 0, cs(stream)>>>(g, cfg->l, n_total, g_ent);
  return launch_status();
}

extern "C" ne_status ne_op_scale(const ne_config* cfg, ne_streams x, int64_t n_total, int64_t s,
                                 const int32_t* g_or_null, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !streams_ok(x, cfg->M)) return NE_EINVAL;
  const int grid = grid_for((n_total + 1) / 2, kThreads);
  NE_DISPATCH_M(cfg->M, k_scale, grid, cs(stream), x, cfg->M, n_total, s, g_or_null);
  return launch_status();
}

extern "C" ne_status ne_op_add(const ne_config* cfg, ne_streams x, ne_cstreams addend, int64_t n_total,
                               int32_t sign, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || (sign != 1 && sign != -1) || !streams_ok(x, cfg->M) || !streams_ok(addend, cfg->M))
    return NE_EINVAL;
  const int grid = grid_for((n_total + 1) / 2, kThreads);
  NE_DISPATCH_M(cfg->M, k_add, grid, cs(stream), x, addend, cfg->M, n_total, sign);
  return launch_status();
}

extern "C" ne_status ne_op_scale_add(const ne_config* cfg, ne_streams x, int64_t n_total, int64_t s,
                                     const int32_t* g_or_null, ne_cstreams addend, int32_t sign, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || (sign != 1 && sign != -1) || !streams_ok(x, cfg->M) || !streams_ok(addend, cfg->M))
    return NE_EINVAL;
  const int grid = grid_for((n_total + 1) / 2, kThreads);
  NE_DISPATCH_M(cfg->M, k_scale_add, grid, cs(stream), x, addend, cfg->M, n_total, s, g_or_null, sign);
  return launch_status();
}

extern "C" ne_status ne_op_outer(const ne_config* cfg, ne_cstreams x, int64_t n1, const int32_t* h,
                                 int64_t n2, ne_streams out, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n1 < 0 || n2 < 0 || !h || !streams_ok(x, cfg->M) || !streams_ok(out, cfg->M)) return NE_EINVAL;
  if (n1 == 0 || n2 == 0) return NE_OK;
  k_outer<<<grid_for((n1 * n2 + 1) / 2, kThreads), kThreads, 0, cs(stream)>>>(x, out, cfg->M, n1, h, n2);
  return launch_status();
}

extern "C" ne_status ne_op_permute(const ne_config* cfg, ne_cstreams x, const int32_t* perm,
                                   int64_t n_total, ne_streams out, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || n_total > INT32_MAX || !perm || !streams_ok(x, cfg->M) || !streams_ok(out, cfg->M))
    return NE_EINVAL;
  NE_DISPATCH_M(cfg->M, k_permute, grid_for(n_total, kThreads), cs(stream), x, out, cfg->M, perm, n_total);
  return launch_status();
}

extern "C" ne_status ne_gen_uniform_i32(uint64_t seed, uint32_t tag, uint32_t gstream, int64_t lo,
                                        int64_t hi, int64_t offset, int64_t count, int32_t* out,
                                        ne_stream_t stream) {
  if (!out || count < 0 || hi <= lo || hi - lo > (1ll << 32) || lo < INT32_MIN || hi - 1 > INT32_MAX)
    return NE_EINVAL;
  if (count == 0) return NE_OK;
  k_gen_uniform<<<grid_for(count, kThreads), kThreads, 0, cs(stream)>>>(ne_gen_key(seed, tag, gstream), lo, hi,
                                                                      offset, count, out);
  return launch_status();
}

extern "C" ne_status ne_gen_perm_i32(uint64_t seed, uint32_t tag, int64_t n, int32_t* out,
                                     ne_stream_t stream) {
  if (!out || n < 0 || n > INT32_MAX) return NE_EINVAL;
  if (n == 0) return NE_OK;
  k_gen_perm<<<grid_for(n, kThreads), kThreads, 0, cs(stream)>>>(ne_gen_key(seed, tag, 0), n, out);
  return launch_status();
}
