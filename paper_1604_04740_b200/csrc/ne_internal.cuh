// ne_internal.cuh — shared device/host helpers of libne (the product path).
// Nothing here is shared with oracle/: this is the CUDA side's own code.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "../../include/ne.h"

namespace ne {

typedef __int128 i128;
typedef unsigned __int128 u128;

constexpr int kThreads = 256;

// ----------------------------------------------------------------- host side
ne_status validate_cfg(const ne_config* cfg);      // M in [3,32], w = 64, Eq. 12
int64_t range_hi(const ne_config* cfg);            // Eq. 13 / Eq. 11 (reading R6)
int num_sms();
int grid_for(int64_t work_items, int threads, int per_sm = 8);
ne_status launch_status();
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline cudaStream_t cs(ne_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// rotate a stream set so that stream r becomes index 0 (the disentangling of
// Eqs. 16-19 depends only on indices relative to r, so the kernels run in the
// rotated frame with r = 0 and write through rotated output pointers)
template <typename S>
inline S rotate(const S& in, int M, int r) {
  S out{};
  for (int j = 0; j < M; ++j) out.s[j] = in.s[(r + j) % M];
  return out;
}

// ----------------------------------------------------------------- device side
__device__ __forceinline__ i128 shl128(i128 x, int s) { return (i128)((u128)x << s); }

// The general form of disentangle_rot below, exact int128 temporaries.
template <int MT, int LT>
__device__ __forceinline__ bool disentangle_rot_i128(const int64_t* e, int M_rt, int l_rt, int64_t* d,
                                                     bool check) {
  const int M = MT > 0 ? MT : M_rt;
  const int l = LT > 0 ? LT : l_rt;
  i128 t = 0;
#pragma unroll
  for (int j = 0; j < (MT > 0 ? MT - 1 : NE_MAX_M - 1); ++j) {
    if (MT == 0 && j > M - 2) break;
    i128 term = shl128((i128)e[1 + j], (M - 2 - j) * l);
    t = (j & 1) ? t - term : t + term;
  }
  if (M & 1) t = -t;
  const int b = (M - 1) * l;  // 1 <= b <= 63 for every valid w = 64 config
  const int64_t dp = (int64_t)((uint64_t)t << (64 - b)) >> (64 - b);
  i128 num = t - (i128)dp;
  if (M & 1) num = -num;
  const i128 dr = num >> b;
  d[0] = (int64_t)dr;
  d[M - 1] = dp;
  i128 prev = dr;
#pragma unroll
  for (int j = 1; j < (MT > 0 ? MT - 1 : NE_MAX_M - 1); ++j) {
    if (MT == 0 && j > M - 2) break;
    i128 cur = (i128)e[j] - shl128(prev, l);
    d[j] = (int64_t)cur;
    prev = cur;
  }
  if (!check) return false;
  return (i128)e[0] != dr + shl128((i128)dp, l);
}

// M = 3 (Eq. 10) in 64-bit registers, bit-identical to the int128 form on
// every input (faulty or not; DESIGN.md §6 "M = 3 check").  With
// t = e2 - 2^l e1 and dp = sext_2l(t):
//   q1 = (dp - e2) / 2^l = (dp >> l) - (e2 >> l)           (dp == e2 mod 2^l)
//   dr = (e1 + q1) / 2^l = (e1 >> l) + (q1 >> l) + [e1 mod 2^l != 0]
// are exact integers of < 2^45, d1 = e1 - 2^l dr is taken mod 2^64, and the
// check e0 == dr + 2^l dp is an exact 2-word compare (|rhs| < 2^66).
template <int LT>
__device__ __forceinline__ bool disentangle3_u64(const int64_t* e, int l_rt, int64_t* d, bool check) {
  const int l = LT > 0 ? LT : l_rt;
  const int b = 2 * l;
  const uint64_t tlo = (uint64_t)e[2] - ((uint64_t)e[1] << l);
  const int64_t dp = (int64_t)(tlo << (64 - b)) >> (64 - b);
  const int64_t q1 = (dp >> l) - (e[2] >> l);
  const int64_t dr = (e[1] >> l) + (q1 >> l) + (((uint64_t)e[1] & ((1ull << l) - 1)) != 0);
  d[0] = dr;
  d[1] = (int64_t)((uint64_t)e[1] - ((uint64_t)dr << l));
  d[2] = dp;
  if (!check) return false;
  const uint64_t lo = (uint64_t)dp << l;
  const uint64_t lo2 = lo + (uint64_t)dr;
  const int64_t hi2 = (dp >> (64 - l)) + (dr >> 63) + (lo2 < lo ? 1 : 0);
  return !(lo2 == (uint64_t)e[0] && hi2 == ((int64_t)lo2 >> 63));
}

// Disentangle + check at one position, in the frame rotated so that the
// excluded stream r is e[0] (Eqs. 16-19 + Eq. 21, readings R1-R4;
// DESIGN.md "disentangle kernel").  e[1..M-1] are the other streams in the
// order (r+1) .. (r+M-1) mod M.  d[j] receives the low 64 bits of d_hat for
// stream (r+j) mod M.  Returns the flag (false when !check).
//   t    = (-1)^M * sum_{j=0}^{M-2} (-1)^j 2^{(M-2-j)l} e[1+j]     (Eq. 16 x (-1)^M)
//   d_p  = sext_{(M-1)l}(t)                      p = M-1              (Eq. 17)
//   d_0  = ((-1)^M (t - d_p)) >> (M-1)l                              (Eq. 18)
//   d_j  = e[j] - 2^l d_{j-1},  j = 1..M-2                           (Eq. 19)
//   flag = e[0] != d_0 + 2^l d_p   (exact, 128-bit)                  (Eq. 21)
// The w = 64 configurations' own l (M = 3: 22, 4: 16, 8: 8) get compile-time
// shift amounts (a uniform branch); M = 3 runs in 64-bit registers.
template <int MT>
__device__ __forceinline__ bool disentangle_rot(const int64_t* e, int M_rt, int l, int64_t* d, bool check) {
  if constexpr (MT == 3) {
    if (l == 22) return disentangle3_u64<22>(e, l, d, check);
    return disentangle3_u64<0>(e, l, d, check);
  } else if constexpr (MT == 4) {
    if (l == 16) return disentangle_rot_i128<4, 16>(e, 4, l, d, check);
    return disentangle_rot_i128<4, 0>(e, 4, l, d, check);
  } else if constexpr (MT == 8) {
    if (l == 8) return disentangle_rot_i128<8, 8>(e, 8, l, d, check);
    return disentangle_rot_i128<8, 0>(e, 8, l, d, check);
  } else {
    return disentangle_rot_i128<MT, 0>(e, M_rt, l, d, check);
  }
}

// Balanced signed base-2^b digits of x, each required to fit int8:
//   d_j = sext_b(x_j) (low b bits, sign-extended), x_{j+1} = (x_j - d_j) >> b,
// exact (x = sum_j d_j 2^(b j)) iff every |d_j| fits int8 and x_L == 0.
// Returns false when x is not representable that way.  (b = 8 is the
// ordinary base-256 split; b = l splits an entangled value c_m + 2^l c_{m-1}
// with |c| < 2^7 into its two int8 halves.)
__device__ __forceinline__ bool digits_b(int64_t x, int b, int L, int8_t* d) {
  bool ok = true;
  for (int j = 0; j < L; ++j) {
    const int64_t dj = (int64_t)((uint64_t)x << (64 - b)) >> (64 - b);
    ok &= (dj >= -128 && dj <= 127);
    d[j] = (int8_t)dj;
    x = (x - dj) >> b;
  }
  return ok && x == 0;
}

// interleave the low 16 bits of x with zeros: bit i -> bit 2i (bitmap words
// of warps that own two consecutive positions per lane)
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// warp-aggregated diagnostics: count + min index, one atomic per warp
__device__ __forceinline__ void diag_add(unsigned long long* count, long long* first, int local_count,
                                         long long local_first) {
  unsigned mask = __ballot_sync(0xffffffffu, local_count != 0);
  if (mask == 0) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    local_count += __shfl_xor_sync(0xffffffffu, local_count, o);
    long long other = __shfl_xor_sync(0xffffffffu, local_first, o);
    local_first = other < local_first ? other : local_first;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(count, (unsigned long long)local_count);
    atomicMin(first, local_first);
  }
}

}  // namespace ne
