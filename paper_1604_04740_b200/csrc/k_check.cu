// k_check.cu — a4 disentangle, a5 reliability check, a6 fail-stop recovery,
// a7 fault injection.  Exact 2w-bit (int128) temporaries on the device
// (footnote P:717-720; a 64-bit compare is not enough).
//
// The host rotates the stream pointers so that the excluded stream r is
// index 0 (ne::rotate); the kernels then run Eqs. 16-19 / Eq. 21 with r = 0
// fully unrolled for M in {3, 4, 8} (generic M through local arrays).
// Streaming layout: every thread owns 2 consecutive positions (one 128-bit
// load/store per stream), a warp owns 64 positions = two bitmap words built
// from two __ballot_sync masks.
#include <cuda_runtime.h>

#include <climits>

#include "ne_internal.cuh"

namespace ne {


template <int MT, bool CHECK>
__global__ void __launch_bounds__(kThreads)
k_disentangle(const __grid_constant__ ne_cstreams e, int M_rt, int l, int64_t n,
              const __grid_constant__ ne_streams d_out, uint32_t* __restrict__ bitmap,
              ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const int64_t npair = (n + 1) / 2;
  const int64_t nwords = (n + 31) / 32;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  int nflag = 0;
  long long first = LLONG_MAX;
  // loop bound rounded up to whole warps so every lane joins the ballots
  const int64_t npair_w = (npair + 31) & ~(int64_t)31;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < npair_w; v += stride) {
    const int64_t n0 = 2 * v;
    bool f0 = false, f1 = false;
    if (n0 < n) {
      const bool pair = n0 + 1 < n;
      int64_t a[MA], b[MA], da[MA], db[MA];
#pragma unroll
      for (int j = 0; j < MA; ++j) {
        if (MT == 0 && j >= M) break;
        if (j == 0 && !CHECK) {
          a[0] = b[0] = 0;
          continue;
        }
        const int64_t* p = e.s[j] + n0;
        if (pair) {
          longlong2 q = __ldcs(reinterpret_cast<const longlong2*>(p));
          a[j] = q.x;
          b[j] = q.y;
        } else {
          a[j] = p[0];
          b[j] = 0;
        }
      }
      f0 = disentangle_rot<MT>(a, M, l, da, CHECK);
      f1 = disentangle_rot<MT>(b, M, l, db, CHECK) && pair;
#pragma unroll
      for (int j = 0; j < MA; ++j) {
        if (MT == 0 && j >= M) break;
        int64_t* q = d_out.s[j] + n0;
        if (pair)
          __stcs(reinterpret_cast<longlong2*>(q), make_longlong2(da[j], db[j]));
        else
          q[0] = da[j];
      }
      if (f0) {
        ++nflag;
        first = n0 < first ? n0 : first;
      }
      if (f1) {
        ++nflag;
        first = (n0 + 1) < first ? (n0 + 1) : first;
      }
    }
    if (CHECK && bitmap) {
      const uint32_t b0 = __ballot_sync(0xffffffffu, f0);
      const uint32_t b1 = __ballot_sync(0xffffffffu, f1);
      const int64_t w0 = (v - lane) / 16;  // 64 positions per warp -> 2 words
      if (lane == 0 && w0 < nwords) bitmap[w0] = spread16(b0) | (spread16(b1) << 1);
      if (lane == 1 && w0 + 1 < nwords) bitmap[w0 + 1] = spread16(b0 >> 16) | (spread16(b1 >> 16) << 1);
    }
  }
  if (CHECK && diag) diag_add(&diag->fault_positions, &diag->first_fault, nflag, first);
}

// Four consecutive positions per thread for M = 3 (the C1 / C3 configs): one
// 256-bit load and store per stream (32-B aligned streams, n % 4 == 0), the
// 64-bit M = 3 disentangle of ne_internal.cuh; a warp owns 128 positions =
// four bitmap words assembled from four ballots.
__device__ __forceinline__ uint32_t word_of4b(const uint32_t (&bal)[4], int j) {
  uint32_t w = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t byte = (bal[u] >> (8 * j)) & 0xffu;
#pragma unroll
    for (int k = 0; k < 8; ++k) w |= ((byte >> k) & 1u) << (4 * k + u);
  }
  return w;
}

template <bool CHECK>
__global__ void __launch_bounds__(kThreads)
k_disentangle3x4(const __grid_constant__ ne_cstreams e, int l, int64_t n, const __grid_constant__ ne_streams d_out,
                 uint32_t* __restrict__ bitmap, ne_diag* __restrict__ diag) {
  const int64_t nq = n / 4;
  const int64_t nwords = (n + 31) / 32;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  int nflag = 0;
  long long first = LLONG_MAX;
  const int64_t nq_w = (nq + 31) & ~(int64_t)31;
  // The check walks the positions from the end (grid-stride sweeps in reverse):
  // the op that produced delta finished with its last tiles, which are still in
  // L2; the recovery pass then walks forward into what the check touched last.
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nsweep = (nq_w + stride - 1) / stride;
  for (int64_t it = 0; it < nsweep; ++it) {
    const int64_t v = (CHECK ? nsweep - 1 - it : it) * stride + tid;
    if (v >= nq_w) continue;  // warp-uniform: nq_w and stride are multiples of 32
    const int64_t n0 = 4 * v;
    bool f[4] = {false, false, false, false};
    if (v < nq) {
      int64_t q[4][3];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (j == 0 && !CHECK) {
          q[0][0] = q[1][0] = q[2][0] = q[3][0] = 0;
          continue;
        }
        uint64_t u0, u1, u2, u3;
        asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(u0), "=l"(u1), "=l"(u2), "=l"(u3)
                     : "l"(e.s[j] + n0));
        q[0][j] = (int64_t)u0; q[1][j] = (int64_t)u1; q[2][j] = (int64_t)u2; q[3][j] = (int64_t)u3;
      }
      int64_t d[4][3];
#pragma unroll
      for (int u = 0; u < 4; ++u) f[u] = disentangle_rot<3>(q[u], 3, l, d[u], CHECK);
#pragma unroll
      for (int j = 0; j < 3; ++j)
        asm volatile("st.global.cs.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(d_out.s[j] + n0), "l"(d[0][j]), "l"(d[1][j]),
                     "l"(d[2][j]), "l"(d[3][j])
                     : "memory");
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
      const int64_t w0 = (v - lane) / 8;
      if (lane < 4 && w0 + lane < nwords) bitmap[w0 + lane] = word_of4b(bal, lane);
    }
  }
  if (CHECK && diag) diag_add(&diag->fault_positions, &diag->first_fault, nflag, first);
}

// a7: exhaustive single-bit sweep.  One warp per trial; lane t owns positions
// 2t, 2t+1 of the window; the flag word is assembled like the bitmap.
template <int MT>
__global__ void __launch_bounds__(kThreads)
k_inject_sweep(const __grid_constant__ ne_cstreams e, int M_rt, int l, int r, int64_t window,
               uint64_t* __restrict__ flagwords, int64_t* __restrict__ dhat) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const int64_t trials = (int64_t)M * window * 64;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < trials; t += nwarps) {
    const int bit = (int)(t & 63);
    const int64_t pos = (t >> 6) % window;
    const int s = (int)((t >> 6) / window);      // original stream index
    const int js = (s - r + M) % M;              // its index in the rotated frame
    bool fl[2] = {false, false};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t p = 2 * lane + h;
      if (p < window) {
        int64_t a[MA], d[MA];
#pragma unroll
        for (int j = 0; j < MA; ++j) {
          if (MT == 0 && j >= M) break;
          a[j] = e.s[j][p];
          if (p == pos && j == js) a[j] ^= (int64_t)(1ull << bit);
        }
        fl[h] = disentangle_rot<MT>(a, M, l, d, true);
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
      const uint64_t lo = spread16(b0) | (spread16(b1) << 1);
      const uint64_t hi = spread16(b0 >> 16) | (spread16(b1 >> 16) << 1);
      flagwords[t] = lo | (hi << 32);
    }
  }
}

__global__ void k_inject(int64_t* x, int64_t idx, uint64_t mask) { x[idx] ^= (int64_t)mask; }

}  // namespace ne

using namespace ne;

template <typename S>
static bool streams_ok(const S& c, int M, int skip = -1) {
  for (int m = 0; m < M; ++m) {
    if (m == skip) continue;
    if (!c.s[m] || !aligned16(c.s[m])) return false;
  }
  return true;
}

template <typename S>
static bool aligned32_all(const S& c, int M, int skip = -1) {
  for (int m = 0; m < M; ++m)
    if (m != skip && (reinterpret_cast<uintptr_t>(c.s[m]) & 31u)) return false;
  return true;
}

template <bool CHECK>
static void launch_disentangle(const ne_config* cfg, const ne_cstreams& er, int64_t n,
                               const ne_streams& dr, uint32_t* bitmap, ne_diag* diag, cudaStream_t s) {
  if (cfg->M == 3 && n % 4 == 0 && aligned32_all(er, 3, CHECK ? -1 : 0) && aligned32_all(dr, 3)) {
    k_disentangle3x4<CHECK><<<grid_for(n / 4, kThreads), kThreads, 0, s>>>(er, cfg->l, n, dr, bitmap, diag);
    return;
  }
  const int grid = grid_for((n + 1) / 2, kThreads);
  switch (cfg->M) {
    case 3: k_disentangle<3, CHECK><<<grid, kThreads, 0, s>>>(er, 3, cfg->l, n, dr, bitmap, diag); break;
    case 4: k_disentangle<4, CHECK><<<grid, kThreads, 0, s>>>(er, 4, cfg->l, n, dr, bitmap, diag); break;
    case 8: k_disentangle<8, CHECK><<<grid, kThreads, 0, s>>>(er, 8, cfg->l, n, dr, bitmap, diag); break;
    default: k_disentangle<0, CHECK><<<grid, kThreads, 0, s>>>(er, cfg->M, cfg->l, n, dr, bitmap, diag); break;
  }
}

extern "C" ne_status ne_disentangle_check(const ne_config* cfg, ne_cstreams delta, int64_t n_total,
                                          int32_t r, ne_streams d_out, uint32_t* bitmap, ne_diag* diag,
                                          ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !streams_ok(delta, cfg->M) || !streams_ok(d_out, cfg->M)) return NE_EINVAL;
  launch_disentangle<true>(cfg, rotate(delta, cfg->M, r), n_total, rotate(d_out, cfg->M, r), bitmap, diag,
                           cs(stream));
  return launch_status();
}

extern "C" ne_status ne_recover(const ne_config* cfg, ne_cstreams delta, int64_t n_total, int32_t r,
                                ne_streams d_out, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  for (int m = 0; m < cfg->M; ++m)
    if (m != r && !delta.s[m]) return NE_EUNRECOVERABLE;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || !streams_ok(delta, cfg->M, r) || !streams_ok(d_out, cfg->M)) return NE_EINVAL;
  launch_disentangle<false>(cfg, rotate(delta, cfg->M, r), n_total, rotate(d_out, cfg->M, r), nullptr, nullptr,
                            cs(stream));
  return launch_status();
}

extern "C" ne_status ne_inject(int64_t* x, int64_t idx, uint64_t mask, ne_stream_t stream) {
  if (!x || idx < 0) return NE_EINVAL;
  k_inject<<<1, 1, 0, cs(stream)>>>(x, idx, mask);
  return launch_status();
}

extern "C" ne_status ne_inject_sweep(const ne_config* cfg, ne_cstreams delta, int64_t window, int32_t r,
                                     uint64_t* flagwords, int64_t* dhat, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  if (window < 1 || window > 64 || !flagwords || !dhat || !streams_ok(delta, cfg->M)) return NE_EINVAL;
  const ne_cstreams er = rotate(delta, cfg->M, r);
  const int64_t trials = (int64_t)cfg->M * window * 64;
  const int grid = grid_for(trials * 32, kThreads);
  cudaStream_t s = cs(stream);
  switch (cfg->M) {
    case 3: k_inject_sweep<3><<<grid, kThreads, 0, s>>>(er, 3, cfg->l, r, window, flagwords, dhat); break;
    case 4: k_inject_sweep<4><<<grid, kThreads, 0, s>>>(er, 4, cfg->l, r, window, flagwords, dhat); break;
    case 8: k_inject_sweep<8><<<grid, kThreads, 0, s>>>(er, 8, cfg->l, r, window, flagwords, dhat); break;
    default: k_inject_sweep<0><<<grid, kThreads, 0, s>>>(er, cfg->M, cfg->l, r, window, flagwords, dhat); break;
  }
  return launch_status();
}
