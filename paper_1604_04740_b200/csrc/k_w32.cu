// k_w32.cu — the paper's own w = 32 instantiation (NEXT-3 of SURVEY §8(f);
// P:528-530 "32-bit integers ... l = 11, k = 10" for M = 3, Table II for the
// rest): entangled streams held in 32-bit containers, which halves the HBM
// bytes of every bandwidth-bound stage relative to w = 64 wherever the
// dynamic range allows (Eq. 11/13: +-1 046 528 for M = 3).
//
// The 2w-bit temporaries of the disentanglement are
// native int64 here: with (M-1) l + k = 32,
//   |t| <= 2^31 sum_j 2^{(M-2-j) l} < 2^63,  b = (M-1) l <= 31,
// so t, d_p = sext_b(t), d_r = (-1)^M (t - d_p) >> b and the check
// e_r == d_r + 2^l d_p are exact in int64; the cascade of Eq. 19 is taken mod
// 2^64 and its low 32 bits stored (the "low w bits" convention, reading R17).
// Layout and vector widths as the w = 64 kernels: 4 positions per thread, one
// 128-bit load/store per stream; a warp covers 128 positions = 4 bitmap words.
#include <cuda_runtime.h>

#include <climits>

#include "ne_internal.cuh"

namespace ne {

// Eqs. 16-19 + 21 in the rotated frame (excluded stream = e[0]), int64 temporaries.
template <int MT>
__device__ __forceinline__ bool disentangle_rot32(const int64_t* e, int M_rt, int l, int32_t* d, bool check) {
  const int M = MT > 0 ? MT : M_rt;
  int64_t t = 0;
#pragma unroll
  for (int j = 0; j < (MT > 0 ? MT - 1 : NE_MAX_M - 1); ++j) {
    if (MT == 0 && j > M - 2) break;
    const int64_t term = (int64_t)((uint64_t)e[1 + j] << ((M - 2 - j) * l));
    t = (j & 1) ? t - term : t + term;
  }
  if (M & 1) t = -t;
  const int b = (M - 1) * l;  // <= 31
  const int64_t dp = (int64_t)((uint64_t)t << (64 - b)) >> (64 - b);
  int64_t num = t - dp;
  if (M & 1) num = -num;
  const int64_t dr = num >> b;
  d[0] = (int32_t)dr;
  d[M - 1] = (int32_t)dp;
  uint64_t prev = (uint64_t)dr;
#pragma unroll
  for (int j = 1; j < (MT > 0 ? MT - 1 : NE_MAX_M - 1); ++j) {
    if (MT == 0 && j > M - 2) break;
    const uint64_t cur = (uint64_t)e[j] - (prev << l);
    d[j] = (int32_t)(uint32_t)cur;
    prev = cur;
  }
  if (!check) return false;
  return e[0] != dr + (int64_t)((uint64_t)dp << l);
}

// bit (4*lane + u) of the warp's 128-position run, from 4 ballots, as word j
__device__ __forceinline__ uint32_t word_of4(const uint32_t (&bal)[4], int j) {
  uint32_t w = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t byte = (bal[u] >> (8 * j)) & 0xffu;
#pragma unroll
    for (int k = 0; k < 8; ++k) w |= ((byte >> k) & 1u) << (4 * k + u);
  }
  return w;
}

template <int MT>
__global__ void __launch_bounds__(kThreads)
k_entangle_w32(const __grid_constant__ ne_cstreams32 c, int M_rt, int l, int64_t hi, int64_t n,
               const __grid_constant__ ne_streams32 eps, ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const int so = blockIdx.y * M;  // stream-set offset (ne_entangle_sets_w32; 0 otherwise)
  int bad = 0;
  long long first = LLONG_MAX;
  const int64_t nv = (n + 3) / 4;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    const bool full = n0 + 3 < n;
    int32_t q[MA][4];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      if (full) {
        const int4 a = __ldcs(reinterpret_cast<const int4*>(c.s[so + m] + n0));
        q[m][0] = a.x; q[m][1] = a.y; q[m][2] = a.z; q[m][3] = a.w;
      } else {
        for (int u = 0; u < 4; ++u) q[m][u] = n0 + u < n ? c.s[so + m][n0 + u] : 0;
      }
    }
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      const int mp = m == 0 ? M - 1 : m - 1;
      int32_t o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        o[u] = (int32_t)((uint32_t)q[m][u] + ((uint32_t)q[mp][u] << l));  // Eq. 15 mod 2^32
        if (n0 + u < n && (q[m][u] > hi || q[m][u] < -hi)) {
          ++bad;
          const long long idx = (long long)(so + m) * n + n0 + u;
          first = idx < first ? idx : first;
        }
      }
      if (full)
        __stcs(reinterpret_cast<int4*>(eps.s[so + m] + n0), make_int4(o[0], o[1], o[2], o[3]));
      else
        for (int u = 0; u < 4; ++u)
          if (n0 + u < n) eps.s[so + m][n0 + u] = o[u];
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// x_m[n] = x_m[n] * (g ? g[n] : s) + sign * a_m[n] (a nullable), mod 2^32:
// the C1 chain's scale and add in one pass (either alone when s = 1 / a = NULL)
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_scale_add_w32(const __grid_constant__ ne_streams32 x, int M_rt, int64_t n, int32_t s, const int32_t* __restrict__ g,
                const __grid_constant__ ne_cstreams32 a, int has_a, int32_t sign) {
  const int M = MT > 0 ? MT : M_rt;
  const int64_t nv = (n + 3) / 4;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = 4 * v;
    const bool full = n0 + 3 < n;
    uint32_t gs[4] = {(uint32_t)s, (uint32_t)s, (uint32_t)s, (uint32_t)s};
    if (g)
      for (int u = 0; u < 4; ++u) gs[u] = n0 + u < n ? (uint32_t)g[n0 + u] : 0u;
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
      uint32_t xv[4], av[4] = {0, 0, 0, 0};
      if (full) {
        const int4 q = *reinterpret_cast<const int4*>(x.s[m] + n0);
        xv[0] = q.x; xv[1] = q.y; xv[2] = q.z; xv[3] = q.w;
        if (has_a) {
          const int4 p = __ldcs(reinterpret_cast<const int4*>(a.s[m] + n0));
          av[0] = p.x; av[1] = p.y; av[2] = p.z; av[3] = p.w;
        }
      } else {
        for (int u = 0; u < 4; ++u) {
          xv[u] = n0 + u < n ? (uint32_t)x.s[m][n0 + u] : 0u;
          if (has_a) av[u] = n0 + u < n ? (uint32_t)a.s[m][n0 + u] : 0u;
        }
      }
      int32_t o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) o[u] = (int32_t)(xv[u] * gs[u] + (uint32_t)sign * av[u]);
      if (full)
        *reinterpret_cast<int4*>(x.s[m] + n0) = make_int4(o[0], o[1], o[2], o[3]);
      else
        for (int u = 0; u < 4; ++u)
          if (n0 + u < n) x.s[m][n0 + u] = o[u];
    }
  }
}

// OP: the C1 op fused in front (delta = x * (g ? g[n] : s) + sign * a, stored
// back to x, then checked from registers; see k_opcheck.cu)
template <int MT, bool CHECK, bool OP = false>
__global__ void __launch_bounds__(kThreads)
k_disentangle_w32(const __grid_constant__ ne_cstreams32 e, int M_rt, int l, int64_t n,
                  const __grid_constant__ ne_streams32 d_out, uint32_t* __restrict__ bitmap,
                  ne_diag* __restrict__ diag, const __grid_constant__ ne_cstreams32 a = ne_cstreams32{},
                  int32_t s = 1, const int32_t* __restrict__ g = nullptr, int32_t sign = 1) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const int64_t nv = (n + 3) / 4;
  const int64_t nwords = (n + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nv_w = (nv + 31) & ~(int64_t)31;  // whole warps join the ballots
  int nflag = 0;
  long long first = LLONG_MAX;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv_w; v += stride) {
    const int64_t n0 = 4 * v;
    bool f[4] = {false, false, false, false};
    if (n0 < n) {
      const bool full = n0 + 3 < n;
      int64_t q[4][MA];
#pragma unroll
      for (int j = 0; j < MA; ++j) {
        if (MT == 0 && j >= M) break;
        if (j == 0 && !CHECK) {
          q[0][0] = q[1][0] = q[2][0] = q[3][0] = 0;
          continue;
        }
        if (full) {
          const int4 v4 = __ldcs(reinterpret_cast<const int4*>(e.s[j] + n0));
          q[0][j] = v4.x; q[1][j] = v4.y; q[2][j] = v4.z; q[3][j] = v4.w;
        } else {
          for (int u = 0; u < 4; ++u) q[u][j] = n0 + u < n ? e.s[j][n0 + u] : 0;
        }
        if (OP) {
          int32_t av[4], gv[4] = {s, s, s, s};
          if (full) {
            const int4 w4 = __ldcs(reinterpret_cast<const int4*>(a.s[j] + n0));
            av[0] = w4.x; av[1] = w4.y; av[2] = w4.z; av[3] = w4.w;
          } else {
            for (int u = 0; u < 4; ++u) av[u] = n0 + u < n ? a.s[j][n0 + u] : 0;
          }
          if (g)
            for (int u = 0; u < 4; ++u) gv[u] = n0 + u < n ? g[n0 + u] : 0;
          int32_t o[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            o[u] = (int32_t)((uint32_t)q[u][j] * (uint32_t)gv[u] + (uint32_t)sign * (uint32_t)av[u]);
            q[u][j] = o[u];
          }
          int32_t* xo = const_cast<int32_t*>(e.s[j]) + n0;
          if (full)
            __stcs(reinterpret_cast<int4*>(xo), make_int4(o[0], o[1], o[2], o[3]));
          else
            for (int u = 0; u < 4; ++u)
              if (n0 + u < n) xo[u] = o[u];
        }
      }
      int32_t d[4][MA];
#pragma unroll
      for (int u = 0; u < 4; ++u) f[u] = disentangle_rot32<MT>(q[u], M, l, d[u], CHECK) && (n0 + u < n);
#pragma unroll
      for (int j = 0; j < MA; ++j) {
        if (MT == 0 && j >= M) break;
        if (full)
          __stcs(reinterpret_cast<int4*>(d_out.s[j] + n0), make_int4(d[0][j], d[1][j], d[2][j], d[3][j]));
        else
          for (int u = 0; u < 4; ++u)
            if (n0 + u < n) d_out.s[j][n0 + u] = d[u][j];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (f[u]) {
          ++nflag;
          first = (n0 + u) < first ? (n0 + u) : first;
        }
    }
    if (CHECK && bitmap) {
      uint32_t bal[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) bal[u] = __ballot_sync(0xffffffffu, f[u]);
      const int64_t w0 = (v - lane) / 8;  // 128 positions per warp -> 4 words
      if (lane < 4 && w0 + lane < nwords) bitmap[w0 + lane] = word_of4(bal, lane);
    }
  }
  if (CHECK && diag) diag_add(&diag->fault_positions, &diag->first_fault, nflag, first);
}

// a7 at w = 32: trial t = (s*window + pos)*32 + bit flips bit `bit` of
// delta_s[pos] and re-runs disentangle + check on positions 0..window-1.
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_inject_sweep_w32(const __grid_constant__ ne_cstreams32 e, int M_rt, int l, int r, int64_t window,
                   uint64_t* __restrict__ flagwords, int32_t* __restrict__ dhat) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const int64_t trials = (int64_t)M * window * 32;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < trials; t += nwarps) {
    const int bit = (int)(t & 31);
    const int64_t pos = (t >> 5) % window;
    const int s = (int)((t >> 5) / window);
    const int js = (s - r + M) % M;
    bool fl[2] = {false, false};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t p = 2 * lane + h;
      if (p < window) {
        int64_t a[MA];
        int32_t d[MA];
#pragma unroll
        for (int j = 0; j < MA; ++j) {
          if (MT == 0 && j >= M) break;
          int32_t v = e.s[j][p];
          if (p == pos && j == js) v ^= (int32_t)(1u << bit);
          a[j] = v;
        }
        fl[h] = disentangle_rot32<MT>(a, M, l, d, true);
        if (p == pos) {
#pragma unroll
          for (int j = 0; j < MA; ++j) {
            if (MT == 0 && j >= M) break;
            dhat[t * M + (r + j) % M] = d[j];
          }
        }
      }
    }
    const uint32_t b0 = __ballot_sync(0xffffffffu, fl[0]);
    const uint32_t b1 = __ballot_sync(0xffffffffu, fl[1]);
    if (lane == 0) {
      uint64_t w = 0;
      for (int k = 0; k < 32; ++k) w |= ((uint64_t)((b0 >> k) & 1u) << (2 * k)) | ((uint64_t)((b1 >> k) & 1u) << (2 * k + 1));
      flagwords[t] = w;
    }
  }
}


// ---- C4 class at w = 32 (NEXT-3: permute + inner where the range allows) ----
// AoS containers x_aos[p * M + m] (int32): with M = 4 one position is 16
// bytes, one 128-bit load in the random gather (half the w = 64 AoS bytes).
template <int MT, bool V4 = false>
__global__ void __launch_bounds__(kThreads)
k_entangle_aos_w32(const __grid_constant__ ne_cstreams32 c, int M_rt, int l, int64_t hi, int64_t n,
                   int32_t* __restrict__ x_aos, ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  int bad = 0;
  long long first = LLONG_MAX;
  if (MT == 4 && V4) {
    // 4 positions per thread: one 128-bit load per stream, four 128-bit stores
    const int64_t nq = n / 4;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
      int32_t cv[4][4];  // [stream][position]
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int4 t = __ldcs(reinterpret_cast<const int4*>(c.s[m]) + q);
        cv[m][0] = t.x; cv[m][1] = t.y; cv[m][2] = t.z; cv[m][3] = t.w;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (cv[m][u] > hi || cv[m][u] < -hi) {
            ++bad;
            const long long idx = (long long)m * n + 4 * q + u;
            first = idx < first ? idx : first;
          }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t e[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) e[m] = (uint32_t)cv[m][u] + ((uint32_t)cv[(m + 3) & 3][u] << l);
        __stcs(reinterpret_cast<uint4*>(x_aos) + 4 * q + u, make_uint4(e[0], e[1], e[2], e[3]));
      }
    }
    if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
    return;
  }
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int32_t cv[MA];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
      if (MT == 0 && m >= M) break;
      cv[m] = __ldcs(c.s[m] + p);
      if (cv[m] > hi || cv[m] < -hi) {
        ++bad;
        const long long idx = (long long)m * n + p;
        first = idx < first ? idx : first;
      }
    }
    uint32_t e[MA];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {  // Eq. 15: eps_m = c_m + 2^l c_{m-1}, mod 2^32
      if (MT == 0 && m >= M) break;
      e[m] = (uint32_t)cv[m] + ((uint32_t)cv[m == 0 ? M - 1 : m - 1] << l);
    }
    if (MT == 4) {
      *reinterpret_cast<uint4*>(x_aos + p * 4) = make_uint4(e[0], e[1], e[2], e[3]);
    } else {
#pragma unroll
      for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
        if (MT == 0 && m >= M) break;
        x_aos[p * M + m] = (int32_t)e[m];
      }
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// permutation gather + blocked inner product + disentangle/check, w = 32:
// one warp per output block, a CTA of 8 warps owns 32 blocks (one bitmap
// word); sums wrap mod 2^32 (the w-bit container arithmetic); the check runs
// Eqs. 16-19 + 21 with int64 temporaries (disentangle_rot32).
constexpr int kPiBlocks = 32, kPiWarps = 8, kPiU = 8;

template <int MT>
__global__ void __launch_bounds__(kPiWarps * 32)
k_pinner_w32(const int32_t* __restrict__ x_aos, int M_rt, int l, const int32_t* __restrict__ perm, int64_t n,
             const int32_t* __restrict__ v, int64_t vlen, int64_t block, const __grid_constant__ ne_streams32 delta_out,
             const __grid_constant__ ne_streams32 d_rot, int r, uint32_t* __restrict__ bitmap,
             ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nb = (n + block - 1) / block;
  __shared__ uint32_t s_flags;
  if (threadIdx.x == 0) s_flags = 0;
  __syncthreads();
  const int64_t b_first = (int64_t)blockIdx.x * kPiBlocks;
  int nflag = 0;
  long long first = LLONG_MAX;
  for (int bi = warp; bi < kPiBlocks; bi += kPiWarps) {
    const int64_t b = b_first + bi;
    if (b >= nb) break;
    const int64_t p_begin = b * block;
    const int64_t p_end = p_begin + block < n ? p_begin + block : n;
    uint32_t acc[MA];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) acc[m] = 0;
    for (int64_t p0 = p_begin + lane; p0 < p_end; p0 += 32 * kPiU) {
      int64_t idx[kPiU];
      uint32_t coef[kPiU];
#pragma unroll
      for (int u = 0; u < kPiU; ++u) {
        const int64_t p = p0 + 32 * u;
        const bool ok = p < p_end;
        idx[u] = ok ? (perm ? (int64_t)__ldcs(perm + p) : p) : -1;
        coef[u] = ok ? (uint32_t)__ldg(v + (vlen == block ? p - p_begin : p % vlen)) : 0u;
      }
      if (MT == 4) {
        uint32_t q[kPiU][4];
#pragma unroll
        for (int u = 0; u < kPiU; ++u) {
          if (idx[u] >= 0) {
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(q[u][0]), "=r"(q[u][1]), "=r"(q[u][2]), "=r"(q[u][3])
                         : "l"(x_aos + idx[u] * 4));
          } else {
            q[u][0] = q[u][1] = q[u][2] = q[u][3] = 0;
          }
        }
#pragma unroll
        for (int u = 0; u < kPiU; ++u)
#pragma unroll
          for (int m = 0; m < 4; ++m) acc[m] += q[u][m] * coef[u];
      } else {
#pragma unroll
        for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
          if (MT == 0 && m >= M) break;
          uint32_t val[kPiU];
#pragma unroll
          for (int u = 0; u < kPiU; ++u) val[u] = idx[u] >= 0 ? (uint32_t)__ldcs(x_aos + idx[u] * M + m) : 0u;
#pragma unroll
          for (int u = 0; u < kPiU; ++u) acc[m] += val[u] * coef[u];
        }
      }
    }
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
      if (MT == 0 && m >= M) break;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[m] += __shfl_xor_sync(0xffffffffu, acc[m], o);
    }
    if (lane == 0) {
      if (delta_out.s[0]) {
#pragma unroll
        for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m) {
          if (MT == 0 && m >= M) break;
          delta_out.s[m][b] = (int32_t)acc[m];
        }
      }
      int64_t e[MA];  // rotated frame: e[j] = delta_{(r+j) mod M}, the w-bit words sign-extended
      int32_t d[MA];
#pragma unroll
      for (int j = 0; j < (MT > 0 ? MT : NE_MAX_M); ++j) {
        if (MT == 0 && j >= M) break;
        int src = r + j;
        if (src >= M) src -= M;
        uint32_t a = 0;
#pragma unroll
        for (int m = 0; m < (MT > 0 ? MT : NE_MAX_M); ++m)
          if (m == src) a = acc[m];
        e[j] = (int64_t)(int32_t)a;
      }
      const bool f = disentangle_rot32<MT>(e, M, l, d, true);
#pragma unroll
      for (int j = 0; j < (MT > 0 ? MT : NE_MAX_M); ++j) {
        if (MT == 0 && j >= M) break;
        d_rot.s[j][b] = d[j];
      }
      if (f) {
        atomicOr(&s_flags, 1u << bi);
        ++nflag;
        first = b < first ? b : first;
      }
    }
  }
  if (diag) diag_add(&diag->fault_positions, &diag->first_fault, nflag, first);
  __syncthreads();
  if (threadIdx.x == 0 && bitmap && b_first < nb) bitmap[blockIdx.x] = s_flags;
}

}  // namespace ne

using namespace ne;

static ne_status validate_cfg32(const ne_config* cfg) {
  if (!cfg) return NE_EINVAL;
  if (cfg->M < 3 || cfg->M > NE_MAX_M || cfg->w != 32) return NE_ECONFIG;
  if (cfg->l < 1 || cfg->k < 1 || cfg->k > cfg->l || (cfg->M - 1) * cfg->l + cfg->k > 32) return NE_ECONFIG;
  return NE_OK;
}

template <typename S>
static bool ok32(const S& c, int M, int skip = -1) {
  for (int m = 0; m < M; ++m) {
    if (m == skip) continue;
    if (!c.s[m] || !aligned16(c.s[m])) return false;
  }
  return true;
}

#define NE_W32_M(M, KERNEL, GRID, STREAM, ...)                             \
  switch (M) {                                                           \
    case 3: KERNEL<3><<<GRID, kThreads, 0, STREAM>>>(__VA_ARGS__); break; \
    case 4: KERNEL<4><<<GRID, kThreads, 0, STREAM>>>(__VA_ARGS__); break; \
    case 8: KERNEL<8><<<GRID, kThreads, 0, STREAM>>>(__VA_ARGS__); break; \
    default: KERNEL<0><<<GRID, kThreads, 0, STREAM>>>(__VA_ARGS__); break; \
  }

extern "C" ne_status ne_entangle_w32(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, ne_streams32 eps,
                                     ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !ok32(c, cfg->M) || !ok32(eps, cfg->M)) return NE_EINVAL;
  NE_W32_M(cfg->M, k_entangle_w32, grid_for((n_total + 3) / 4, kThreads), cs(stream), c, cfg->M, cfg->l,
           range_hi(cfg), n_total, eps, diag);
  return launch_status();
}

extern "C" ne_status ne_entangle_sets_w32(const ne_config* cfg, ne_cstreams32 c, int32_t sets, int64_t n_total,
                                          ne_streams32 eps, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  if (sets < 1 || sets * cfg->M > NE_MAX_M) return NE_EINVAL;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !ok32(c, sets * cfg->M) || !ok32(eps, sets * cfg->M)) return NE_EINVAL;
  const dim3 grid((unsigned)grid_for((n_total + 3) / 4, kThreads, (8 + sets - 1) / sets), (unsigned)sets);
  NE_W32_M(cfg->M, k_entangle_w32, grid, cs(stream), c, cfg->M, cfg->l, range_hi(cfg), n_total, eps, diag);
  return launch_status();
}

extern "C" ne_status ne_op_scale_add_w32(const ne_config* cfg, ne_streams32 x, int64_t n_total, int32_t s,
                                         const int32_t* g_or_null, const ne_cstreams32* addend_or_null, int32_t sign,
                                         ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || (sign != 1 && sign != -1) || !ok32(x, cfg->M)) return NE_EINVAL;
  ne_cstreams32 a{};
  if (addend_or_null) {
    if (!ok32(*addend_or_null, cfg->M)) return NE_EINVAL;
    a = *addend_or_null;
  }
  NE_W32_M(cfg->M, k_scale_add_w32, grid_for((n_total + 3) / 4, kThreads), cs(stream), x, cfg->M, n_total, s,
           g_or_null, a, addend_or_null ? 1 : 0, sign);
  return launch_status();
}

template <bool CHECK>
static void launch_dis32(const ne_config* cfg, const ne_cstreams32& er, int64_t n, const ne_streams32& dr,
                         uint32_t* bitmap, ne_diag* diag, cudaStream_t s) {
  const int grid = grid_for((n + 3) / 4, kThreads);
  switch (cfg->M) {
    case 3: k_disentangle_w32<3, CHECK><<<grid, kThreads, 0, s>>>(er, 3, cfg->l, n, dr, bitmap, diag); break;
    case 4: k_disentangle_w32<4, CHECK><<<grid, kThreads, 0, s>>>(er, 4, cfg->l, n, dr, bitmap, diag); break;
    case 8: k_disentangle_w32<8, CHECK><<<grid, kThreads, 0, s>>>(er, 8, cfg->l, n, dr, bitmap, diag); break;
    default: k_disentangle_w32<0, CHECK><<<grid, kThreads, 0, s>>>(er, cfg->M, cfg->l, n, dr, bitmap, diag); break;
  }
}

extern "C" ne_status ne_disentangle_check_w32(const ne_config* cfg, ne_cstreams32 delta, int64_t n_total, int32_t r,
                                              ne_streams32 d_out, uint32_t* bitmap, ne_diag* diag,
                                              ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !ok32(delta, cfg->M) || !ok32(d_out, cfg->M)) return NE_EINVAL;
  launch_dis32<true>(cfg, rotate(delta, cfg->M, r), n_total, rotate(d_out, cfg->M, r), bitmap, diag, cs(stream));
  return launch_status();
}

extern "C" ne_status ne_recover_w32(const ne_config* cfg, ne_cstreams32 delta, int64_t n_total, int32_t r,
                                    ne_streams32 d_out, ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  for (int m = 0; m < cfg->M; ++m)
    if (m != r && !delta.s[m]) return NE_EUNRECOVERABLE;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !ok32(delta, cfg->M, r) || !ok32(d_out, cfg->M)) return NE_EINVAL;
  launch_dis32<false>(cfg, rotate(delta, cfg->M, r), n_total, rotate(d_out, cfg->M, r), nullptr, nullptr, cs(stream));
  return launch_status();
}

extern "C" ne_status ne_op_scale_add_check_w32(const ne_config* cfg, ne_streams32 x, int64_t n_total, int32_t s,
                                               const int32_t* g_or_null, ne_cstreams32 addend, int32_t sign, int32_t r,
                                               ne_streams32 d_out, uint32_t* bitmap, ne_diag* diag,
                                               ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || (sign != 1 && sign != -1) || !ok32(x, cfg->M) || !ok32(addend, cfg->M) || !ok32(d_out, cfg->M))
    return NE_EINVAL;
  ne_cstreams32 xc{};
  for (int m = 0; m < cfg->M; ++m) xc.s[m] = x.s[m];
  const ne_cstreams32 xr = rotate(xc, cfg->M, r), ar = rotate(addend, cfg->M, r);
  const ne_streams32 dr = rotate(d_out, cfg->M, r);
  const int grid = grid_for((n_total + 3) / 4, kThreads);
  cudaStream_t cst = cs(stream);
  switch (cfg->M) {
    case 3: k_disentangle_w32<3, true, true><<<grid, kThreads, 0, cst>>>(xr, 3, cfg->l, n_total, dr, bitmap, diag, ar, s, g_or_null, sign); break;
    case 4: k_disentangle_w32<4, true, true><<<grid, kThreads, 0, cst>>>(xr, 4, cfg->l, n_total, dr, bitmap, diag, ar, s, g_or_null, sign); break;
    case 8: k_disentangle_w32<8, true, true><<<grid, kThreads, 0, cst>>>(xr, 8, cfg->l, n_total, dr, bitmap, diag, ar, s, g_or_null, sign); break;
    default: k_disentangle_w32<0, true, true><<<grid, kThreads, 0, cst>>>(xr, cfg->M, cfg->l, n_total, dr, bitmap, diag, ar, s, g_or_null, sign); break;
  }
  return launch_status();
}

extern "C" ne_status ne_inject_sweep_w32(const ne_config* cfg, ne_cstreams32 delta, int64_t window, int32_t r,
                                         uint64_t* flagwords, int32_t* dhat, ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  if (window < 1 || window > 64 || !flagwords || !dhat || !ok32(delta, cfg->M)) return NE_EINVAL;
  const int64_t trials = (int64_t)cfg->M * window * 32;
  NE_W32_M(cfg->M, k_inject_sweep_w32, grid_for(trials * 32, kThreads), cs(stream), rotate(delta, cfg->M, r), cfg->M,
           cfg->l, r, window, flagwords, dhat);
  return launch_status();
}

extern "C" ne_status ne_entangle_aos_w32(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t* x_aos,
                                         ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !ok32(c, cfg->M) || !x_aos || !aligned16(x_aos)) return NE_EINVAL;
  cudaStream_t s = cs(stream);
  if (cfg->M == 4 && n_total % 4 == 0) {  // streams 16-B aligned (ok32): vectorised form
    k_entangle_aos_w32<4, true><<<grid_for(n_total / 4, kThreads), kThreads, 0, s>>>(c, 4, cfg->l, range_hi(cfg),
                                                                                     n_total, x_aos, diag);
    return launch_status();
  }
  const int grid = grid_for(n_total, kThreads);
  NE_W32_M(cfg->M, k_entangle_aos_w32, grid, s, c, cfg->M, cfg->l, range_hi(cfg), n_total, x_aos, diag);
  return launch_status();
}

extern "C" ne_status ne_op_permute_inner_check_w32(const ne_config* cfg, const int32_t* x_aos, const int32_t* perm,
                                                   int64_t n_total, const int32_t* v, int64_t vlen, int64_t block,
                                                   int32_t r, ne_streams32 delta_out, ne_streams32 d_out,
                                                   uint32_t* bitmap, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg32(cfg);
  if (st != NE_OK) return st;
  const int M = cfg->M;
  if (r < 0 || r >= M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || n_total > INT32_MAX || block < 1 || vlen < 1 || !v || !x_aos || !aligned16(x_aos) ||
      !ok32(d_out, M))
    return NE_EINVAL;
  if (delta_out.s[0] && !ok32(delta_out, M)) return NE_EINVAL;
  const int64_t nb = (n_total + block - 1) / block;
  const int grid = (int)((nb + kPiBlocks - 1) / kPiBlocks);
  const ne_streams32 drot = rotate(d_out, M, r);
  cudaStream_t s = cs(stream);
  switch (M) {
    case 3: k_pinner_w32<3><<<grid, kPiWarps * 32, 0, s>>>(x_aos, M, cfg->l, perm, n_total, v, vlen, block, delta_out, drot, r, bitmap, diag); break;
    case 4: k_pinner_w32<4><<<grid, kPiWarps * 32, 0, s>>>(x_aos, M, cfg->l, perm, n_total, v, vlen, block, delta_out, drot, r, bitmap, diag); break;
    case 8: k_pinner_w32<8><<<grid, kPiWarps * 32, 0, s>>>(x_aos, M, cfg->l, perm, n_total, v, vlen, block, delta_out, drot, r, bitmap, diag); break;
    default: k_pinner_w32<0><<<grid, kPiWarps * 32, 0, s>>>(x_aos, M, cfg->l, perm, n_total, v, vlen, block, delta_out, drot, r, bitmap, diag); break;
  }
  return launch_status();
}
