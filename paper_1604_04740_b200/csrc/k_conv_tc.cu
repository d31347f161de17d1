// k_conv_tc.cu — circular convolution / cross-correlation of the entangled
// streams on the tensor cores (NEXT-2 of SURVEY §8(f)): the direct form
// (reading R12)
//     out_m[n] = sum_{j<T} g[j] eps_m[(n - j) mod N]        (conv)
//     out_m[n] = sum_{j<T} g[j] eps_m[(n + j) mod N]        (correlation)
// written as a Toeplitz GEMM.  Output block b = outputs W b .. W b + W-1
// (W = 128, or 256 for long kernels with <= 2 digit planes: conv_block):
//     out_m[W b + i] = sum_{k<Kpad} W_b[k] G[i][k],
//     W_b[k] = eps_m[(W b + k - s0) mod N],   s0 = T - 1 (conv) or 0 (corr),
//     G[i][k] = g[i + s0 - k] (conv) or g[k - i] (corr), 0 outside [0, T),
// with Kpad = roundup(T + W - 1, 128).  eps_m is held as L int8 digit planes
// (the GEMM's digit plan), circularly extended so that window
// row b is the contiguous bytes [W b, W b + Kpad) of each plane:
//     plane_{m,d}[t] = digit d of eps_m[(t - s0) mod N],  0 <= t < plane_len.
// The GEMM is k_gemm_tc in Toeplitz mode (rows = blocks, cols = W, K = Kpad,
// B = G); every D_{m,d} G product is exact in int32 (Kpad * 2^14 < 2^31) and
// recombined in int64.  The last N mod W outputs (a partial block) are
// computed by k_conv_tail from the same planes.  Redundancy: Kpad / T MACs
// per useful MAC (4x at T = 64, 1.08x at T = 4500 with W = 256), paid on a
// pipe ~100x faster than the IMAD path of k_conv.cu.
#include <cuda_runtime.h>

#include <climits>

#include "ne_internal.cuh"

namespace ne {

ne_status launch_conv_tc(int M, int L, int b, int W, const int8_t* planes, int64_t plane_rows, const int8_t* Gt,
                         int64_t Kpad, int64_t nblocks, const ne_streams& C, cudaStream_t s);

// output block width W (= GEMM columns): 256 when the taps are long enough
// that the extra W - 1 window bytes cost little (T >= 256) and TMEM holds the
// L limb accumulators of a 256-wide tile (L <= 2); 128 otherwise
static int conv_block(int64_t taps, int L) { return (taps >= 256 && L <= 2) ? 256 : 128; }
static int64_t conv_kpad(int64_t taps, int W) { return (taps + W - 1 + 127) / 128 * 128; }
static int64_t conv_plane_len(int64_t n, int64_t taps, int W) {
  const int64_t nb_all = (n + W - 1) / W;
  return (W * nb_all + conv_kpad(taps, W) + W - 1) / W * W;
}

// a1 into circularly extended digit planes: 4 consecutive t per thread, all M
// streams in order (each c_m[n] read once per t, used by streams m and m+1).
// Three restructurings were A/B-measured slower or equal on one box (C2P,
// N = 10^6, T = 4500, M = 8 / 3: 18.0 / 10.2 us here): one aligned 128-bit
// load per lane with a funnel shift across lanes (22.2 / 12.4), every
// stream's loads issued before any store (18.2 / 9.9), one thread per
// (stream, quad) (20.5 / 11.3); r02z52 (base 16.5 / 10.2 that box): stream
// m + 1's loads issued before stream m is digitised 18.5 / 10.5, a one-wave
// grid of 148 x 4 CTAs 18.7 / 10.5, both 20.6 / 12.1.  r02z54: warp-coalesced loads (lane
// loads t0 + lane + 32 u, digit bytes re-packed through a per-warp shared
// row) 18.6 / 10.7 vs 16.6 / 10.3 (parity green, dropped).  The kernel costs ~6 us fixed + ~1.5 us per
// stream: a launch-latency-dominated pass of 6 MB per stream.
// The range assertion (a0) counts every position once: t in [s0, s0 + N).
#ifndef NE_CP_MINB  // >= 4 CTAs per SM (<= 64 registers): r02 A/B (scripts/r02/z41.sh), M = 8 / 3:
#define NE_CP_MINB 4  // 1 (76 regs) 18.2 / 11.1 us, 4 (58) 17.6 / 10.0, 6 (40, spills) 18.6 / 11.5, 8 (32) 20.1 / 12.0
#endif
template <int MT>
__global__ void __launch_bounds__(kThreads, NE_CP_MINB)
k_entangle_conv_planes(const __grid_constant__ ne_cstreams32 c, int M_rt, int l, int64_t hi, int64_t n, int64_t s0,
                       int64_t s0mod, int64_t plane_len, int L, int b, int8_t* __restrict__ planes,
                       ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const bool pair = L == 2 && b == l && b <= 31;
  (void)MA;
  int bad = 0;
  long long first = LLONG_MAX;
  const int64_t nq = plane_len / 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    // position of t = 4q: (t - s0) mod n without a 64-bit division
    // (s0mod = s0 mod n; t - s0mod < plane_len, a few multiples of n at most)
    int64_t p = 4 * q - s0mod;
    if (p < 0) p += n;
    while (p >= n) p -= n;
    int64_t pos[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      pos[u] = p;
      if (++p == n) p = 0;
    }
    // which of the 4 t are counted by the range assertion (t in [s0, s0 + N))
    bool tin[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) tin[u] = 4 * q + u >= s0 && 4 * q + u < s0 + n;
    // streams in order with only the previous one live (registers: the M = 8
    // instantiation stays at full occupancy); c_{M-1} first, the "previous"
    // stream of stream 0 (circulant Eq. 14)
    int32_t prv[4], cur[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) prv[u] = __ldg(c.s[M - 1] + pos[u]);
#pragma unroll 1
    for (int m = 0; m < M; ++m) {
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = __ldg(c.s[m] + pos[u]);
      uint32_t w[4] = {0, 0, 0, 0};
      unsigned badm = 0;  // bit u: position u out of range / not representable
      if (pair) {
        // the two-digit base-2^l plan in 32-bit arithmetic (as k_entangle_pair):
        // d0 = sext_b(c), d1 = c_prev + (c >> b) + bit_{b-1}(c); packed 4 bytes at a time
        int32_t d0[4], d1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          d0[u] = (int32_t)((uint32_t)cur[u] << (32 - b)) >> (32 - b);
          d1[u] = prv[u] + (cur[u] >> b) + ((cur[u] >> (b - 1)) & 1);
          const bool out = ((uint32_t)(d0[u] + 128) | (uint32_t)(d1[u] + 128)) > 255u ||
                           (hi < INT32_MAX && (cur[u] > hi || cur[u] < -hi));
          badm |= (unsigned)out << u;
        }
        w[0] = __byte_perm(__byte_perm(d0[0], d0[1], 0x0040), __byte_perm(d0[2], d0[3], 0x0040), 0x5410);
        w[1] = __byte_perm(__byte_perm(d1[0], d1[1], 0x0040), __byte_perm(d1[2], d1[3], 0x0040), 0x5410);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t cc = cur[u];
          const int64_t x = (int64_t)((uint64_t)cc + ((uint64_t)(int64_t)prv[u] << l));
          int8_t d[4];
          const bool ok = digits_b(x, b, L, d);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < L) w[j] |= (uint32_t)(uint8_t)d[j] << (8 * u);
          badm |= (unsigned)(cc > hi || cc < -hi || !ok) << u;
        }
      }
      if (badm) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (((badm >> u) & 1) && tin[u]) {
            ++bad;
            const long long idx = (long long)m * n + pos[u];
            first = idx < first ? idx : first;
          }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < L) __stcs(reinterpret_cast<unsigned int*>(planes + ((int64_t)m * L + j) * plane_len + 4 * q), w[j]);
#pragma unroll
      for (int u = 0; u < 4; ++u) prv[u] = cur[u];
    }
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// ABFT comparison (NEXT-1 on the conv, Eqs. 3-5): plain data as one int8
// digit per stream and the checksum stream r = sum_m c_m (Eq. 4) as Ls
// balanced base-256 digits, in the same circularly extended plane layout, one
// pass; values that do not fit are range violations (data: m*N + n; checksum:
// M*N + n), each position counted once.
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_abft_conv_planes(const __grid_constant__ ne_cstreams32 c, int M_rt, int64_t n, int64_t s0, int64_t s0mod,
                   int64_t plane_len, int Ls, int8_t* __restrict__ pdata, int8_t* __restrict__ psum,
                   ne_diag* __restrict__ diag) {
  const int M = MT > 0 ? MT : M_rt;
  int bad = 0;
  long long first = LLONG_MAX;
  const int64_t nq = plane_len / 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = 4 * q - s0mod;
    if (p < 0) p += n;
    while (p >= n) p -= n;
    int64_t pos[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      pos[u] = p;
      if (++p == n) p = 0;
    }
    int64_t sum[4] = {0, 0, 0, 0};
#pragma unroll 1
    for (int m = 0; m < M; ++m) {
      uint32_t w = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t v = __ldg(c.s[m] + pos[u]);
        sum[u] += v;
        w |= (uint32_t)(uint8_t)(int8_t)v << (8 * u);
        const int64_t t = 4 * q + u;
        if (t >= s0 && t < s0 + n && (v < -128 || v > 127)) {
          ++bad;
          const long long idx = (long long)m * n + pos[u];
          first = idx < first ? idx : first;
        }
      }
      __stcs(reinterpret_cast<unsigned int*>(pdata + (int64_t)m * plane_len + 4 * q), w);
    }
    uint32_t ws[4] = {0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int8_t d[4];
      const bool ok = digits_b(sum[u], 8, Ls, d);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < Ls) ws[j] |= (uint32_t)(uint8_t)d[j] << (8 * u);
      const int64_t t = 4 * q + u;
      if (t >= s0 && t < s0 + n && !ok) {
        ++bad;
        const long long idx = (long long)M * n + pos[u];
        first = idx < first ? idx : first;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < Ls) __stcs(reinterpret_cast<unsigned int*>(psum + (int64_t)j * plane_len + 4 * q), ws[j]);
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// G (W x Kpad int8, K contiguous): conv G[i][k] = g[i + T - 1 - k],
// correlation G[i][k] = g[k - i]; taps outside [-128, 127] are range
// violations (counted once per tap, first_bad = tap index).
__global__ void __launch_bounds__(kThreads)
k_conv_prep_taps(const int32_t* __restrict__ g, int64_t T, int correlate, int64_t Kpad, int8_t* __restrict__ Gt,
                 ne_diag* __restrict__ diag) {
  int bad = 0;
  long long first = LLONG_MAX;
  const int64_t i = blockIdx.y;  // row of G (output within the block)
  for (int64_t k4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 4 * k4 < Kpad; k4 += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = 4 * k4 + u;
      const int64_t j = correlate ? k - i : i + T - 1 - k;
      const int32_t v = (j >= 0 && j < T) ? __ldg(g + j) : 0;
      w |= (uint32_t)(uint8_t)(int8_t)v << (8 * u);
      if (i == 0 && k < T) {  // tap k checked once
        const int32_t gk = __ldg(g + k);
        if (gk < -128 || gk > 127) {
          ++bad;
          first = k < first ? k : first;
        }
      }
    }
    *reinterpret_cast<uint32_t*>(Gt + i * Kpad + 4 * k4) = w;
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// the last n - W nb outputs of every stream (a partial block): one CTA of
// 128 threads per output, threads split k in 16-byte pieces (4 dp4a each),
// exact int32 digit sums (Kpad 2^14 < 2^31) reduced by shuffles and shared
// memory, recombined in int64
__global__ void __launch_bounds__(128)
k_conv_tail(const int8_t* __restrict__ planes, int M, int L, int b, int64_t plane_len, const int8_t* __restrict__ Gt,
            int64_t Kpad, int64_t nb, int W, int64_t n, const __grid_constant__ ne_streams out) {
  __shared__ int32_t part[4][4];
  const int64_t tail = n - (int64_t)W * nb;
  const int m = (int)(blockIdx.x / tail);
  const int64_t i = blockIdx.x % tail;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int4* g = reinterpret_cast<const int4*>(Gt + i * Kpad);  // Kpad % 128 == 0: 16-byte aligned rows
  for (int d = 0; d < L; ++d) {
    const int4* w = reinterpret_cast<const int4*>(planes + ((int64_t)m * L + d) * plane_len + (int64_t)W * nb);
    int32_t s = 0;
#pragma unroll 4
    for (int64_t k = threadIdx.x; k < Kpad / 16; k += 128) {
      const int4 x = __ldg(w + k), y = __ldg(g + k);
      s = __dp4a(x.x, y.x, s);
      s = __dp4a(x.y, y.y, s);
      s = __dp4a(x.z, y.z, s);
      s = __dp4a(x.w, y.w, s);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) part[d][wp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int d = 0; d < L; ++d)
      acc += (uint64_t)(int64_t)(part[d][0] + part[d][1] + part[d][2] + part[d][3]) << (b * d);
    out.s[m][(int64_t)W * nb + i] = (int64_t)acc;
  }
}

}  // namespace ne

using namespace ne;

extern "C" ne_status ne_conv_geometry(int64_t n_total, int32_t taps, int32_t L, int32_t* block, int64_t* kpad,
                                      int64_t* plane_len) {
  if (n_total < 1 || taps < 1 || L < 1 || L > 4 || !block || !kpad || !plane_len) return NE_EINVAL;
  *block = conv_block(taps, L);
  *kpad = conv_kpad(taps, *block);
  *plane_len = conv_plane_len(n_total, taps, *block);
  return NE_OK;
}

extern "C" ne_status ne_entangle_limbs_conv(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t taps,
                                            int32_t correlate, int32_t L, int32_t limb_bits, int32_t block,
                                            int8_t* planes, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total < 1 || taps < 1 || (correlate != 0 && correlate != 1) || L < 1 || L > 4 || limb_bits < 8 ||
      limb_bits > 63 || (block != 128 && block != 256) || !planes || !aligned16(planes))
    return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (!c.s[m]) return NE_EINVAL;
  const int64_t plen = conv_plane_len(n_total, taps, block);
  const int64_t s0 = correlate ? 0 : (int64_t)taps - 1;
  const int64_t s0m = s0 % n_total;
  const int grid = grid_for(plen / 4, kThreads);
  cudaStream_t s = cs(stream);
  const int64_t hi = range_hi(cfg);
  switch (cfg->M) {
    case 3: k_entangle_conv_planes<3><<<grid, kThreads, 0, s>>>(c, 3, cfg->l, hi, n_total, s0, s0m, plen, L, limb_bits, planes, diag); break;
    case 4: k_entangle_conv_planes<4><<<grid, kThreads, 0, s>>>(c, 4, cfg->l, hi, n_total, s0, s0m, plen, L, limb_bits, planes, diag); break;
    case 8: k_entangle_conv_planes<8><<<grid, kThreads, 0, s>>>(c, 8, cfg->l, hi, n_total, s0, s0m, plen, L, limb_bits, planes, diag); break;
    default: k_entangle_conv_planes<0><<<grid, kThreads, 0, s>>>(c, cfg->M, cfg->l, hi, n_total, s0, s0m, plen, L, limb_bits, planes, diag); break;
  }
  return launch_status();
}

extern "C" ne_status ne_conv_prep_taps(const int32_t* g, int32_t taps, int32_t correlate, int32_t block, int8_t* Gt,
                                       ne_diag* diag, ne_stream_t stream) {
  if (!g || taps < 1 || (correlate != 0 && correlate != 1) || (block != 128 && block != 256) || !Gt ||
      !aligned16(Gt))
    return NE_EINVAL;
  const int64_t kp = conv_kpad(taps, block);
  const dim3 grid((unsigned)((kp / 4 + kThreads - 1) / kThreads), (unsigned)block);
  k_conv_prep_taps<<<grid, kThreads, 0, cs(stream)>>>(g, taps, correlate, kp, Gt, diag);
  return launch_status();
}

extern "C" ne_status ne_op_conv_limbs(const ne_config* cfg, const int8_t* planes, int32_t L, int32_t limb_bits,
                                      int32_t block, const int8_t* Gt, int64_t n_total, int32_t taps,
                                      int32_t correlate, ne_streams out, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total < 1 || taps < 1 || (correlate != 0 && correlate != 1) || L < 1 || L > 4 || limb_bits < 8 ||
      limb_bits > 63 || (block != 128 && block != 256) || !planes || !Gt || !aligned16(planes) || !aligned16(Gt))
    return NE_EINVAL;
  if (block == 256 && L > 2) return NE_ENOTSUP;  // 256-wide tiles hold at most 2 limb accumulators in TMEM
  const int64_t kp = conv_kpad(taps, block);
  if (kp >= 131072) return NE_ENOTSUP;  // int32 digit sums stay exact: Kpad * 128 * 128 < 2^31
  for (int m = 0; m < cfg->M; ++m)
    if (!out.s[m] || !aligned16(out.s[m])) return NE_EINVAL;
  const int64_t plen = conv_plane_len(n_total, taps, block);
  const int64_t nb = n_total / block;
  cudaStream_t s = cs(stream);
  if (nb > 0 && (st = launch_conv_tc(cfg->M, L, limb_bits, block, planes, plen / block, Gt, kp, nb, out, s)) != NE_OK)
    return st;
  const int64_t tail = n_total - (int64_t)block * nb;
  if (tail > 0)
    k_conv_tail<<<(unsigned)(cfg->M * tail), 128, 0, s>>>(planes, cfg->M, L, limb_bits, plen, Gt, kp, nb, block,
                                                          n_total, out);
  return launch_status();
}

extern "C" ne_status ne_abft_encode_conv(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t taps,
                                         int32_t correlate, int32_t block, int8_t* pdata, int32_t Ls, int8_t* psum,
                                         ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total < 1 || taps < 1 || (correlate != 0 && correlate != 1) || (block != 128 && block != 256) || Ls < 1 ||
      Ls > 4 || !pdata || !psum || !aligned16(pdata) || !aligned16(psum))
    return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    if (!c.s[m]) return NE_EINVAL;
  const int64_t plen = conv_plane_len(n_total, taps, block);
  const int64_t s0 = correlate ? 0 : (int64_t)taps - 1;
  const int grid = grid_for(plen / 4, kThreads);
  cudaStream_t s = cs(stream);
  switch (cfg->M) {
    case 3: k_abft_conv_planes<3><<<grid, kThreads, 0, s>>>(c, 3, n_total, s0, s0 % n_total, plen, Ls, pdata, psum, diag); break;
    case 8: k_abft_conv_planes<8><<<grid, kThreads, 0, s>>>(c, 8, n_total, s0, s0 % n_total, plen, Ls, pdata, psum, diag); break;
    default: k_abft_conv_planes<0><<<grid, kThreads, 0, s>>>(c, cfg->M, n_total, s0, s0 % n_total, plen, Ls, pdata, psum, diag); break;
  }
  return launch_status();
}

extern "C" ne_status ne_op_conv_limbs_plain(int32_t count, const int8_t* planes, int32_t L, int32_t limb_bits,
                                            int32_t block, const int8_t* Gt, int64_t n_total, int32_t taps,
                                            int32_t correlate, ne_streams out, ne_stream_t stream) {
  if (count < 1 || count > 8 || n_total < 1 || taps < 1 || (correlate != 0 && correlate != 1) || L < 1 || L > 4 ||
      limb_bits < 8 || limb_bits > 63 || (block != 128 && block != 256) || !planes || !Gt || !aligned16(planes) ||
      !aligned16(Gt))
    return NE_EINVAL;
  if (block == 256 && L > 2) return NE_ENOTSUP;
  const int64_t kp = conv_kpad(taps, block);
  if (kp >= 131072) return NE_ENOTSUP;
  for (int m = 0; m < count; ++m)
    if (!out.s[m] || !aligned16(out.s[m])) return NE_EINVAL;
  const int64_t plen = conv_plane_len(n_total, taps, block);
  const int64_t nb = n_total / block;
  cudaStream_t s = cs(stream);
  ne_status st;
  if (nb > 0 && (st = launch_conv_tc(count, L, limb_bits, block, planes, plen / block, Gt, kp, nb, out, s)) != NE_OK)
    return st;
  const int64_t tail = n_total - (int64_t)block * nb;
  if (tail > 0)
    k_conv_tail<<<(unsigned)(count * tail), 128, 0, s>>>(planes, count, L, limb_bits, plen, Gt, kp, nb, block, n_total,
                                                        out);
  return launch_status();
}

