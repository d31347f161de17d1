// k_opcheck.cu — LSB ops with the disentangle + check (a4/a5) fused into the
// op's own kernel (BASELINE north star: "the entangle, extract and check
// stages are fused into the producer and consumer kernels wherever the
// operation allows").  Each kernel computes delta_m = eps_m op g for ALL M
// streams of its positions — every stream's value from that stream's operand
// only, so a fault in one stream's computation still corrupts one delta_m and
// is caught (Props 2/4) — stores delta (it is what a later fail-stop recovery
// reads), then runs Eqs. 16-19 + 21 on the values it holds and writes d_hat,
// the fault bitmap and ne_diag exactly as k_disentangle<M, true> would from
// the stored delta.  Bit-identical to op + ne_disentangle_check.
//   k_scale_add_check : delta = eps * (g ? g[n] : s) + sign * alpha (C1 chain)
//   k_conv_check      : direct circular conv / correlation (reading R12),
//                       all M streams of a 256 P-output tile per CTA (C2)
// The entangle stays a separate pass: entangling on load would let one fault
// in a plain value corrupt two streams consistently.
#include <cuda_runtime.h>

#include <climits>

#include "ne_internal.cuh"

namespace ne {

template <int MT>
__global__ void __launch_bounds__(kThreads)
k_scale_add_check(const __grid_constant__ ne_streams x, const __grid_constant__ ne_cstreams a, int l, int64_t n,
                  int64_t s, const int32_t* __restrict__ g, int sign, const __grid_constant__ ne_streams d_out,
                  uint32_t* __restrict__ bitmap, ne_diag* __restrict__ diag) {
  const int64_t npair = (n + 1) / 2;
  const int64_t nwords = (n + 31) / 32;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const uint64_t sg = (uint64_t)(int64_t)sign;
  int nflag = 0;
  long long first = LLONG_MAX;
  const int64_t npair_w = (npair + 31) & ~(int64_t)31;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < npair_w; v += stride) {
    const int64_t n0 = 2 * v;
    bool f0 = false, f1 = false;
    if (n0 < n) {
      const bool pair = n0 + 1 < n;
      uint64_t fa = (uint64_t)s, fb = (uint64_t)s;
      if (g) {
        fa = (uint64_t)(int64_t)g[n0];
        fb = pair ? (uint64_t)(int64_t)g[n0 + 1] : 0;
      }
      int64_t da[MT], db[MT], ra[MT], rb[MT];
      if (pair) {
        // (issuing every stream's loads before any store measured slower at
        // 2^27: 2.172 vs 2.124 ms, scripts/r02/ab.py --case c1_sac)
#pragma unroll
        for (int j = 0; j < MT; ++j) {
          const longlong2 u = __ldcs(reinterpret_cast<const longlong2*>(x.s[j] + n0));
          const longlong2 w = __ldcs(reinterpret_cast<const longlong2*>(a.s[j] + n0));
          da[j] = (int64_t)((uint64_t)u.x * fa + sg * (uint64_t)w.x);
          db[j] = (int64_t)((uint64_t)u.y * fb + sg * (uint64_t)w.y);
          __stcs(reinterpret_cast<longlong2*>(x.s[j] + n0), make_longlong2(da[j], db[j]));
        }
      } else {
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        int64_t* p = x.s[j] + n0;
        const int64_t* q = a.s[j] + n0;
        {
          da[j] = (int64_t)((uint64_t)p[0] * fa + sg * (uint64_t)q[0]);
          db[j] = 0;
          p[0] = da[j];
        }
      }
      }
      f0 = disentangle_rot<MT>(da, MT, l, ra, true);
      f1 = disentangle_rot<MT>(db, MT, l, rb, true) && pair;
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        int64_t* q = d_out.s[j] + n0;
        if (pair)
          __stcs(reinterpret_cast<longlong2*>(q), make_longlong2(ra[j], rb[j]));
        else
          q[0] = ra[j];
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
    if (bitmap) {
      const uint32_t b0 = __ballot_sync(0xffffffffu, f0);
      const uint32_t b1 = __ballot_sync(0xffffffffu, f1);
      const int64_t w0 = (v - lane) / 16;
      if (lane == 0 && w0 < nwords) bitmap[w0] = spread16(b0) | (spread16(b1) << 1);
      if (lane == 1 && w0 + 1 < nwords) bitmap[w0 + 1] = spread16(b0 >> 16) | (spread16(b1 >> 16) << 1);
    }
  }
  if (diag) diag_add(&diag->fault_positions, &diag->first_fault, nflag, first);
}

// Direct conv of all MT streams over a tile of 256 * P outputs; taps in chunks
// of kTCc staged in shared memory together with the circular windows of ALL
// MT streams (one load phase, one barrier per chunk: the windows' L2/DRAM
// latencies overlap instead of adding up stream by stream); the int32-window
// fast path of k_conv.cu (IMAD.WIDE) when every window fits int32, the full
// 64-bit MAC otherwise.  Thread t owns outputs n0 + t + 256 p, so a warp's 32
// consecutive outputs are one bitmap word.  (r02 A/B: splitting the streams
// over thread groups — 256 x M threads per block, one stream per thread, two
// accumulators — to raise occupancy at C2's 256 blocks measured slower: C2
// 10.0 -> 15.8 us, M = 3 T = 1000 54.7 -> 134.6 us; the per-output form
// shares each tap load over M MACs.  Late r02: 64 threads x 4 consecutive
// outputs per tile with the window sliding through registers (a quarter of
// the shared loads) measured slower too — C2 9.9 -> 14.3 us, M = 8 19.0 ->
// 34.2, T = 300 22.2 -> 34.6 (scripts/r02/z49.sh): the tile's window load,
// spread over 4x fewer threads, is what the kernel waits on.)
constexpr int kTCc = 256;

template <int MT, int P>
constexpr size_t conv_check_smem() {
  return (size_t)MT * (256 * P + kTCc) * 12 + (size_t)kTCc * 4;
}

template <int MT, int P>
__global__ void __launch_bounds__(256)
k_conv_check(const __grid_constant__ ne_cstreams x, const __grid_constant__ ne_streams out, int64_t N,
             const int32_t* __restrict__ g, int T, int correlate, int l, const __grid_constant__ ne_streams d_out,
             uint32_t* __restrict__ bitmap, ne_diag* __restrict__ diag) {
  constexpr int TILE = 256 * P;
  constexpr int WS = TILE + kTCc;  // window slots per stream
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* xs = reinterpret_cast<int64_t*>(smem);            // [MT][WS]
  int32_t* xs32 = reinterpret_cast<int32_t*>(xs + MT * WS);  // [MT][WS]
  int32_t* gs = xs32 + MT * WS;                              // [kTCc]
  const int64_t n0 = (int64_t)blockIdx.x * TILE;
  int64_t acc[MT][P];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int p = 0; p < P; ++p) acc[m][p] = 0;

  for (int j0 = 0; j0 < T; j0 += kTCc) {
    const int tc = T - j0 < kTCc ? T - j0 : kTCc;
    const int wlen = TILE + tc - 1;
    for (int j = threadIdx.x; j < tc; j += 256) gs[j] = __ldg(g + j0 + j);
    int64_t base = correlate ? (n0 + j0) : (n0 - j0 - (tc - 1));
    base %= N;
    if (base < 0) base += N;
    int fits = 1;
#ifndef NE_CONV_WLOAD2  // r02 A/B (scripts/r02/z50.sh): C2 10.1 -> 9.9 us, M = 8 18.8 -> 18.0, T = 300 equal
#define NE_CONV_WLOAD2 1
#endif
    if (NE_CONV_WLOAD2 && wlen <= 512) {
      // every stream's (at most two) window values loaded before any is stored: one load latency
      int64_t v[MT][2];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int q = threadIdx.x + 256 * k;
          int64_t idx = base + q;
          if (idx >= N) idx %= N;
          v[m][k] = q < wlen ? __ldg(x.s[m] + idx) : 0;
        }
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int q = threadIdx.x + 256 * k;
          if (q < wlen) {
            xs[m * WS + q] = v[m][k];
            xs32[m * WS + q] = (int32_t)v[m][k];
            fits &= (v[m][k] == (int64_t)(int32_t)v[m][k]);
          }
        }
    } else {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        for (int q = threadIdx.x; q < wlen; q += 256) {
          int64_t idx = base + q;
          if (idx >= N) idx %= N;
          const int64_t val = __ldg(x.s[m] + idx);
          xs[m * WS + q] = val;
          xs32[m * WS + q] = (int32_t)val;
          fits &= (val == (int64_t)(int32_t)val);
        }
      }
    }
    fits = __syncthreads_and(fits);
    if (fits) {
      for (int j = 0; j < tc; ++j) {
        const int64_t gj = gs[j];
        const int off = correlate ? j : (tc - 1 - j);
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int p = 0; p < P; ++p)
            acc[m][p] = (int64_t)((uint64_t)acc[m][p] + (uint64_t)(gj * (int64_t)xs32[m * WS + threadIdx.x + 256 * p + off]));
      }
    } else {
      for (int j = 0; j < tc; ++j) {
        const uint64_t gj = (uint64_t)(int64_t)gs[j];
        const int off = correlate ? j : (tc - 1 - j);
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int p = 0; p < P; ++p)
            acc[m][p] = (int64_t)((uint64_t)acc[m][p] + gj * (uint64_t)xs[m * WS + threadIdx.x + 256 * p + off]);
      }
    }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  int nflag = 0;
  long long first = LLONG_MAX;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int64_t n = n0 + threadIdx.x + 256 * p;
    bool f = false;
    if (n < N) {
      int64_t e[MT], d[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        e[m] = acc[m][p];
        __stcs(out.s[m] + n, e[m]);
      }
      f = disentangle_rot<MT>(e, MT, l, d, true);
#pragma unroll
      for (int m = 0; m < MT; ++m) __stcs(d_out.s[m] + n, d[m]);
      if (f) {
        ++nflag;
        first = n < first ? n : first;
      }
    }
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if (bitmap && lane == 0 && n - lane < N) bitmap[(n - lane) / 32] = b;
  }
  if (diag) diag_add(&diag->fault_positions, &diag->first_fault, nflag, first);
}

}  // namespace ne

using namespace ne;

template <typename S>
static bool all_ok(const S& c, int M) {
  for (int m = 0; m < M; ++m)
    if (!c.s[m] || !aligned16(c.s[m])) return false;
  return true;
}

extern "C" ne_status ne_op_scale_add_check(const ne_config* cfg, ne_streams x, int64_t n_total, int64_t s,
                                           const int32_t* g_or_null, ne_cstreams addend, int32_t sign, int32_t r,
                                           ne_streams d_out, uint32_t* bitmap, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || (sign != 1 && sign != -1) || !all_ok(x, cfg->M) || !all_ok(addend, cfg->M) ||
      !all_ok(d_out, cfg->M))
    return NE_EINVAL;
  cudaStream_t cst = cs(stream);
  const int grid = grid_for((n_total + 1) / 2, kThreads);
  const ne_streams xr = rotate(x, cfg->M, r), dr = rotate(d_out, cfg->M, r);
  const ne_cstreams ar = rotate(addend, cfg->M, r);
  switch (cfg->M) {
    case 3: k_scale_add_check<3><<<grid, kThreads, 0, cst>>>(xr, ar, cfg->l, n_total, s, g_or_null, sign, dr, bitmap, diag); break;
    case 4: k_scale_add_check<4><<<grid, kThreads, 0, cst>>>(xr, ar, cfg->l, n_total, s, g_or_null, sign, dr, bitmap, diag); break;
    case 8: k_scale_add_check<8><<<grid, kThreads, 0, cst>>>(xr, ar, cfg->l, n_total, s, g_or_null, sign, dr, bitmap, diag); break;
    default: {  // other M: the two kernels back to back (same results)
      if ((st = ne_op_scale_add(cfg, x, n_total, s, g_or_null, addend, sign, stream)) != NE_OK) return st;
      ne_cstreams xc{};
      for (int m = 0; m < cfg->M; ++m) xc.s[m] = x.s[m];
      return ne_disentangle_check(cfg, xc, n_total, r, d_out, bitmap, diag, stream);
    }
  }
  return launch_status();
}

template <int MT, int P>
static void launch_conv_check(const ne_config* cfg, const ne_cstreams& xr, int64_t n, const int32_t* g, int taps,
                              int correlate, const ne_streams& outr, const ne_streams& dr, uint32_t* bitmap,
                              ne_diag* diag, cudaStream_t s) {
  constexpr size_t smem = conv_check_smem<MT, P>();
  cudaFuncSetAttribute(k_conv_check<MT, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned grid = (unsigned)((n + 256 * P - 1) / (256 * P));
  k_conv_check<MT, P><<<grid, 256, smem, s>>>(xr, outr, n, g, taps, correlate, cfg->l, dr, bitmap, diag);
}

extern "C" ne_status ne_op_conv_check(const ne_config* cfg, ne_cstreams x, int64_t n_total, const int32_t* g,
                                      int32_t taps, int32_t correlate, ne_streams out, int32_t r, ne_streams d_out,
                                      uint32_t* bitmap, ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (r < 0 || r >= cfg->M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || taps < 1 || !g || (correlate != 0 && correlate != 1) || !all_ok(x, cfg->M) ||
      !all_ok(out, cfg->M) || !all_ok(d_out, cfg->M))
    return NE_EINVAL;
  for (int m = 0; m < cfg->M; ++m)
    for (int q = 0; q < cfg->M; ++q)
      if ((const void*)x.s[q] == (const void*)out.s[m]) return NE_EINVAL;  // out must not alias x
  cudaStream_t s = cs(stream);
  const ne_cstreams xr = rotate(x, cfg->M, r);
  const ne_streams outr = rotate(out, cfg->M, r), dr = rotate(d_out, cfg->M, r);
  switch (cfg->M) {
    case 3: launch_conv_check<3, 1>(cfg, xr, n_total, g, taps, correlate, outr, dr, bitmap, diag, s); break;
    case 4: launch_conv_check<4, 1>(cfg, xr, n_total, g, taps, correlate, outr, dr, bitmap, diag, s); break;
    case 8: launch_conv_check<8, 1>(cfg, xr, n_total, g, taps, correlate, outr, dr, bitmap, diag, s); break;
    default: {
      if ((st = ne_op_conv(cfg, x, n_total, g, taps, correlate, out, stream)) != NE_OK) return st;
      ne_cstreams oc{};
      for (int m = 0; m < cfg->M; ++m) oc.s[m] = out.s[m];
      return ne_disentangle_check(cfg, oc, n_total, r, d_out, bitmap, diag, stream);
    }
  }
  return launch_status();
}
