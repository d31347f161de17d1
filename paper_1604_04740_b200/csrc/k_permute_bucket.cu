// k_permute_bucket.cu — the fused permutation + blocked inner product of C4 as
// a partitioned scatter-reduce: no random DRAM gather (the C4 default).
//
// The op (P:253-258 permutation, then the blocked inner product of Eq. 2):
//   delta_m[b] = sum_{i in block b} x_m[perm[i]] * v[i mod vlen]
// The gather form (k_inner.cu, k_pinner) reads x at random positions: every
// 32-byte AoS entry costs a 128-byte DRAM line fill (profiles/r02_c4_floor.md).
// Here the pairs (i, perm[i]) are partitioned into cells (w, d): w = the
// source window perm[i] >> S (2^S entries of x, a slice of L2), d = the
// destination range of RB output blocks that i falls in (RB x M int64 sums
// fit one CTA's shared memory).  Cells are laid out window-major.
//   pass 1 (k_pb_scatter): per chunk of consecutive i (one d per chunk), the
//     pairs sorted by w in shared memory and written to their cells (one
//     atomic per (chunk, w) reserves the slice); cells have a fixed capacity
//     (mean + 8 sigma of a random permutation's cell sizes): pairs past it go
//     to an overflow list (skewed permutations; k_pb_overflow adds them with
//     global 64-bit reductions after pass 2);
//   pass 2 (k_pb_reduce): CTA d walks its cells w = 0, 1, ... in window order
//     (all CTAs move through x window by window, so the window being read is
//     in L2), gathers x[perm[i]] from L2, and adds the M products with
//     v[i mod vlen] into its shared-memory block sums (two independent 32-bit
//     shared atomics per product: its low 20 bits and the rest; a soft
//     lockstep keeps the CTAs within two windows), then adds its RB blocks
//     into delta (zeroed) once;
//   then ne_disentangle_check on delta, exactly as the gather path.
// Measured (profiles/r02_c4_bucket.md, r02c_ncu_summary.md): C4 stage 5.20 ms
// vs 5.80 ms for the gather kernel; every line of x fetched once (10.8 GB for
// pairs + x against 35.2 GB); the reduce bound by its shared atomics.
// Every sum is an int64 sum mod 2^64, so delta is bit-identical to the gather
// order (wrap-free for certified results).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "ne_internal.cuh"

namespace ne {

#ifndef NE_PB_CHUNK
#define NE_PB_CHUNK 4096  // (r02 A/B: 4096 / 512 threads 5.06 ms, 8192 / 512 5.12, 4096 / 256 5.21, 16384 / 1024 5.17)
#endif
#ifndef NE_PB_STHREADS
#define NE_PB_STHREADS 512
#endif
constexpr int kPbChunk = NE_PB_CHUNK;       // positions per scatter CTA (one destination range)
constexpr int kPbSThreads = NE_PB_STHREADS; // scatter threads
constexpr int kPbThreads = 512;             // reduce threads
constexpr int kPbMaxWin = 1024;     // windows
constexpr int kPbAccBytes = 32768;  // shared block sums per reduce CTA
constexpr int kPbU = 4;             // pairs per reduce thread and iteration (strided by the CTA)

struct PbGeo {
  int S;          // window shift
  int nwin;       // windows
  int64_t rb;     // output blocks per destination range
  int64_t span;   // positions per destination range (rb * block)
  int nrange;     // destination ranges
  int64_t chunks_per_range;
  int64_t cells;  // nwin * nrange
  int64_t cap;    // pair slots per cell (mean + 8 sigma + 32); the rest overflow
};

static PbGeo pb_geo(int64_t n, int M, int64_t block) {
  PbGeo g{};
  int S = 21;
  int64_t budget = 32ll << 20;
  if (const char* e = getenv("NE_PB_WINDOW_MB")) budget = atoll(e) << 20;  // experiments
  while (S > 4 && (int64_t)M * 8 << S > budget) --S;  // window of x <= 32 MB (r02: best of 16-64)
  while (S > 4 && (n >> S) < 16) --S;
  while (((n + (1ll << S) - 1) >> S) > kPbMaxWin) ++S;
  g.S = S;
  g.nwin = (int)((n + (1ll << S) - 1) >> S);
  const int64_t nb = (n + block - 1) / block;
  // destination ranges: two reduce CTAs per SM (uniform progress through the
  // windows), at most the shared-memory block sums of one CTA
  g.rb = std::max<int64_t>(1, std::min<int64_t>(kPbAccBytes / (8 * M), (nb + 2 * num_sms() - 1) / (2 * num_sms())));
  g.span = g.rb * block;
  g.nrange = (int)((nb + g.rb - 1) / g.rb);
  g.chunks_per_range = (std::min<int64_t>(g.span, n) + kPbChunk - 1) / kPbChunk;
  g.cells = (int64_t)g.nwin * g.nrange;
  const int64_t mu = (n + g.cells - 1) / g.cells;
  g.cap = (mu + 8 * (int64_t)ceil(sqrt((double)mu)) + 32 + 3) / 4 * 4;
  return g;
}

// chunk c of destination range d: positions [d span + c kPbChunk, ... ) clipped to the range and n
__device__ __forceinline__ void pb_chunk(int64_t n, int64_t span, int64_t cpr, int64_t& c0, int& len, int& d) {
  d = (int)(blockIdx.x / cpr);
  const int64_t lo = (int64_t)d * span + (blockIdx.x % cpr) * kPbChunk;
  const int64_t hi = min(min((int64_t)(d + 1) * span, lo + kPbChunk), n);
  c0 = lo;
  len = (int)max((int64_t)0, hi - lo);
}

__global__ void __launch_bounds__(kPbSThreads)
k_pb_scatter(const int32_t* __restrict__ perm, int64_t n, int S, int nwin, int64_t span, int64_t cpr, int nrange,
             int64_t cap, unsigned* __restrict__ fill, int2* __restrict__ pairs, unsigned* __restrict__ ovn,
             int2* __restrict__ ov, ne_diag* __restrict__ diag) {
  extern __shared__ __align__(16) unsigned char smem[];
  int2* buf = reinterpret_cast<int2*>(smem);                    // [kPbChunk]
  unsigned* cnt = reinterpret_cast<unsigned*>(buf + kPbChunk);  // [kPbMaxWin]
  unsigned* off = cnt + kPbMaxWin;                              // [kPbMaxWin] chunk-local offsets
  unsigned* gbase = off + kPbMaxWin;                            // [kPbMaxWin] first slot in the cell
  int64_t c0;
  int len, d;
  pb_chunk(n, span, cpr, c0, len, d);
  for (int w = threadIdx.x; w < nwin; w += kPbSThreads) cnt[w] = 0;
  __syncthreads();
  constexpr int kPer = kPbChunk / kPbSThreads;
  int32_t jv[kPer];
  unsigned rk[kPer];
  int bad = 0;
  long long first = LLONG_MAX;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int k = u * kPbSThreads + threadIdx.x;
    jv[u] = k < len ? __ldcs(perm + c0 + k) : -1;
    if (k < len && (jv[u] < 0 || jv[u] >= n)) {  // not a permutation of [0, n): counted, skipped
      ++bad;
      first = c0 + k < first ? c0 + k : first;
      jv[u] = -1;
    }
    if (jv[u] >= 0) rk[u] = atomicAdd(&cnt[jv[u] >> S], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // chunk-local exclusive scan over windows (one warp, 32 at a time)
    const int lane = threadIdx.x;
    unsigned carry = 0;
    for (int w0 = 0; w0 < nwin; w0 += 32) {
      const unsigned c = w0 + lane < nwin ? cnt[w0 + lane] : 0u;
      unsigned x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (w0 + lane < nwin) off[w0 + lane] = carry + x - c;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  for (int w = threadIdx.x; w < nwin; w += kPbSThreads) {
    const int64_t cell = (int64_t)w * nrange + d;
    gbase[w] = cnt[w] ? atomicAdd(&fill[cell], cnt[w]) : 0u;   // this chunk's slice of the cell
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int k = u * kPbSThreads + threadIdx.x;
    if (k < len && jv[u] >= 0) buf[off[jv[u] >> S] + rk[u]] = make_int2((int32_t)(c0 + k), jv[u]);
  }
  __syncthreads();
  const unsigned total = off[nwin - 1] + cnt[nwin - 1];
  for (unsigned k = threadIdx.x; k < total; k += kPbSThreads) {
    const int2 p = buf[k];
    const int w = p.y >> S;
    const int64_t r = (int64_t)gbase[w] + (k - off[w]);
    if (r < cap)
      pairs[((int64_t)w * nrange + d) * cap + r] = p;
    else
      ov[atomicAdd(ovn, 1u)] = p;   // a cell past its capacity (skewed permutations): the overflow list
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// the overflow list: pairs whose cell was full, added into delta with global
// 64-bit reductions (any order: every pass adds into the zeroed delta)
template <int MT>
__global__ void __launch_bounds__(256)
k_pb_overflow(const int64_t* __restrict__ x_aos, int M_rt, const int2* __restrict__ ov, const unsigned* __restrict__ ovn,
              int32_t block, const int32_t* __restrict__ v, int32_t vlen, ne_streams delta) {
  const int M = MT > 0 ? MT : M_rt;
  const unsigned cnt = *ovn;
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
    const int2 pr = ov[k];
    const uint64_t wgt = (uint64_t)(int64_t)__ldg(v + pr.x % vlen);
    const int b = pr.x / block;
    for (int m = 0; m < M; ++m) {
      const uint64_t p = (uint64_t)x_aos[(int64_t)pr.y * M + m] * wgt;
      asm volatile("red.global.add.u64 [%0], %1;" ::"l"(delta.s[m] + b), "l"(p) : "memory");
    }
  }
}

template <int MT>
__global__ void __launch_bounds__(kPbThreads, 2)  // two per SM: every reduce CTA resident (the window lockstep)
k_pb_reduce(const int64_t* __restrict__ x_aos, int M_rt, const int2* __restrict__ pairs,
            const unsigned* __restrict__ fill, int64_t cap, unsigned* __restrict__ done,
            int nwin, int nrange, int64_t rb, int32_t block, const int32_t* __restrict__ v, int32_t vlen, int64_t nb,
            int lockstep, int fast, ne_streams delta) {
  constexpr int MA = MT > 0 ? MT : 8;  // M <= 8 (host check)
  const int M = MT > 0 ? MT : M_rt;
  // block sums as two 32-bit words per (block, stream): a product p with
  // |p| < 2^40 adds its low 20 bits (unsigned) into word 0 and p >> 20
  // (signed, |.| <= 2^20) into word 1 — two independent native 32-bit shared
  // atomics (a 64-bit shared atomicAdd is a CAS loop on this target); with at
  // most 2048 products per block neither word can overflow (fast != 0), and
  // the block sum is word1 * 2^20 + word0.  Any other product is added
  // straight into delta (zeroed; red.add.u64), as are the CTA's sums at the end.
  __shared__ unsigned acc[kPbAccBytes / 4];  // [rb][M][2]
  const int d = blockIdx.x;
  const int64_t b0 = (int64_t)d * rb;
  for (int k = threadIdx.x; k < rb * M * 2; k += kPbThreads) acc[k] = 0;
  __syncthreads();
  for (int w = 0; w < nwin; ++w) {
    // soft lockstep: start window w only when every CTA has finished window
    // w - 2, so at most ~3 windows of x are being read at any time (all CTAs
    // resident: checked on the host)
    if (lockstep && w >= 2) {
      if (threadIdx.x == 0) {  // bounded: the lockstep only buys locality, never correctness
        for (int spin = 0; spin < (1 << 20) && *(volatile unsigned*)(done + w - 2) < (unsigned)nrange; ++spin)
          __nanosleep(100);
      }
      __syncthreads();
    }
    const int64_t cell = (int64_t)w * nrange + d;
    const int64_t lo = cell * cap;
    const unsigned cnt = (unsigned)min((int64_t)fill[cell], cap);
    // kPbU pairs per thread and iteration (strided: coalesced pair loads),
    // their x entries in flight together
    for (unsigned k0 = threadIdx.x; k0 < cnt; k0 += kPbU * kPbThreads) {
      int2 pr[kPbU];
#pragma unroll
      for (int u = 0; u < kPbU; ++u) {
        const unsigned k = k0 + u * kPbThreads;
        pr[u] = k < cnt ? __ldcs(pairs + lo + k) : make_int2(-1, 0);
      }
      uint64_t c[kPbU][MA];
      int64_t wg[kPbU];
#pragma unroll
      for (int u = 0; u < kPbU; ++u) {
        if (pr[u].x < 0) continue;
        wg[u] = __ldg(v + pr[u].x % vlen);
        const int64_t* xe = x_aos + (int64_t)pr[u].y * M;
        if (MT == 4) {
          uint64_t u0, u1, u2, u3;
          asm("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(u0), "=l"(u1), "=l"(u2), "=l"(u3) : "l"(xe));
          c[u][0] = u0; c[u][1] = u1; c[u][2] = u2; c[u][3] = u3;
        } else {
#pragma unroll
          for (int m = 0; m < (MT > 0 ? MT : M); ++m) c[u][m] = (uint64_t)__ldg(xe + m);
        }
      }
#pragma unroll
      for (int u = 0; u < kPbU; ++u) {
        if (pr[u].x < 0) continue;
        const int bl = (int)(pr[u].x / block - b0);
#pragma unroll
        for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
          const uint64_t p = c[u][m] * (uint64_t)wg[u];
          if (fast && p + (1ull << 40) < (1ull << 41)) {
            unsigned* a = acc + 2 * (bl * M + m);
            atomicAdd(a, (unsigned)p & 0xFFFFFu);
            atomicAdd(a + 1, (unsigned)(int)((int64_t)p >> 20));
          } else {
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(delta.s[m] + b0 + bl), "l"(p) : "memory");
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(done + w, 1u);
  }
  __syncthreads();
  const int64_t nbl = min(rb, nb - b0);
  for (int64_t k = threadIdx.x; k < nbl * M; k += kPbThreads) {
    const int64_t bl = k / M;
    const int m = (int)(k % M);
    const uint64_t sum = (uint64_t)((int64_t)(int)acc[2 * k + 1] * (1ll << 20)) + (uint64_t)acc[2 * k];
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(delta.s[m] + b0 + bl), "l"(sum) : "memory");
  }
}

static bool pb_streams_ok(const ne_streams& c, int M) {
  for (int m = 0; m < M; ++m)
    if (!c.s[m] || !aligned16(c.s[m])) return false;
  return true;
}

}  // namespace ne

using namespace ne;

extern "C" ne_status ne_permute_inner_workspace(const ne_config* cfg, int64_t n_total, int64_t block,
                                                size_t* bytes) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!bytes || n_total < 0 || n_total > INT32_MAX || block < 1) return NE_EINVAL;
  const PbGeo g = pb_geo(std::max<int64_t>(n_total, 1), cfg->M, block);
  // cells at fixed capacity, an overflow list as long as the input (any bijection fits), the fill
  // counters, the overflow count and the window counters
  *bytes = ((size_t)g.cells * g.cap + (size_t)std::max<int64_t>(n_total, 1)) * sizeof(int2) +
           ((size_t)g.cells + 1 + g.nwin) * sizeof(unsigned) + 256;
  return NE_OK;
}

extern "C" ne_status ne_op_permute_inner_check_bucketed(const ne_config* cfg, const int64_t* x_aos,
                                                        const int32_t* perm, int64_t n_total, const int32_t* v,
                                                        int64_t vlen, int64_t block, int32_t r, ne_streams delta,
                                                        ne_streams d_out, uint32_t* bitmap, ne_diag* diag,
                                                        void* workspace, size_t ws_bytes, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  const int M = cfg->M;
  if (r < 0 || r >= M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || n_total > INT32_MAX || block < 1 || block > INT32_MAX || vlen < 1 || vlen > INT32_MAX || !v ||
      !perm || !x_aos || !aligned16(x_aos) || !pb_streams_ok(delta, M) || !pb_streams_ok(d_out, M) || !workspace ||
      !aligned16(workspace))
    return NE_EINVAL;
  if (M > 8) return NE_ENOTSUP;
  size_t need = 0;
  ne_permute_inner_workspace(cfg, n_total, block, &need);
  if (ws_bytes < need) return NE_EINVAL;
  const PbGeo g = pb_geo(n_total, M, block);
  const int64_t nb = (n_total + block - 1) / block;
  cudaStream_t s = cs(stream);
  int2* pairs = static_cast<int2*>(workspace);
  int2* ov = pairs + g.cells * g.cap;
  unsigned* fill = reinterpret_cast<unsigned*>(ov + n_total);
  unsigned* ovn = fill + g.cells;
  unsigned* done = ovn + 1;
  if (cudaMemsetAsync(fill, 0, ((size_t)g.cells + 1 + g.nwin) * sizeof(unsigned), s) != cudaSuccess) return NE_ECUDA;
  for (int m = 0; m < M; ++m)  // every pass adds into delta
    if (cudaMemsetAsync(delta.s[m], 0, (size_t)nb * sizeof(int64_t), s) != cudaSuccess) return NE_ECUDA;
  const unsigned nchunk = (unsigned)(g.nrange * g.chunks_per_range);
  const size_t smem = (size_t)kPbChunk * sizeof(int2) + 3 * kPbMaxWin * sizeof(unsigned);
  cudaFuncSetAttribute(k_pb_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_pb_scatter<<<nchunk, kPbSThreads, smem, s>>>(perm, n_total, g.S, g.nwin, g.span, g.chunks_per_range, g.nrange,
                                                g.cap, fill, pairs, ovn, ov, diag);
  // the window lockstep needs every reduce CTA resident at once
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pb_reduce<4>, kPbThreads, 0) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 0;
  }
  const int lockstep = g.nrange <= (int64_t)per_sm * num_sms() ? 1 : 0;
#define NE_PB_RED(MV)                                                                                             \
  k_pb_reduce<MV><<<g.nrange, kPbThreads, 0, s>>>(x_aos, M, pairs, fill, g.cap, done, g.nwin, g.nrange, g.rb,    \
                                                  (int32_t)block, v, (int32_t)vlen, nb, lockstep, block <= 2048,  \
                                                  delta);                                                         \
  k_pb_overflow<MV><<<num_sms(), 256, 0, s>>>(x_aos, M, ov, ovn, (int32_t)block, v, (int32_t)vlen, delta)
  switch (M) {
    case 4: NE_PB_RED(4); break;
    case 3: NE_PB_RED(3); break;
    case 8: NE_PB_RED(8); break;
    default: NE_PB_RED(0); break;
  }
#undef NE_PB_RED
  if ((st = launch_status()) != NE_OK) return st;
  ne_cstreams dc{};
  for (int m = 0; m < M; ++m) dc.s[m] = delta.s[m];
  return ne_disentangle_check(cfg, dc, nb, r, d_out, bitmap, diag, stream);
}
