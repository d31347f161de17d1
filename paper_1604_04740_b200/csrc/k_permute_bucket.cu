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
// Owned-run mode (mode 1 of ne_permute_inner_plan, the C4 default; below
// k_pb_overflow): chunk slices sorted by (window, block) so each block's
// pairs form one run per cell, 32-bit pairs, a run index per (cell, block),
// and a reduce without atomics — each block owned by one thread, cells staged
// in shared memory by TMA, x gathered through L2 only: C4 stage 3.9 ms.
// Every sum is an int64 sum mod 2^64, so delta is bit-identical to the gather
// order (wrap-free for certified results).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "ne_internal.cuh"
#include "tc_common.cuh"

#ifndef NE_PB_XLD
#define NE_PB_XLD "ld.global.cg.v4.u64"  // the gathered x entry (32 B, M = 4), cached in L2 only
#endif

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
#ifdef NE_PB_OWN_OFF
constexpr bool kPbOwnOff = true;  // A/B builds: the shared-atomic reduce everywhere
#else
constexpr bool kPbOwnOff = false;
#endif
#ifndef NE_PO_LAG
#define NE_PO_LAG 2
#endif
constexpr int kPoLag = NE_PO_LAG;  // own: a CTA starts window w once every CTA finished w - kPoLag
constexpr size_t kPoSmemMax = 224 * 1024;  // own: reduce shared memory (block sums + two staged cells)
constexpr int kPoAccBytes = 128 * 1024;  // own: block sums per reduce CTA (owner-only int64, shared memory)
#ifndef NE_PO_THREADS
#define NE_PO_THREADS 1024
#endif
constexpr int kPoMaxThreads = NE_PO_THREADS;  // own: reduce threads (at most)

struct PbGeo {
  int S;          // window shift
  int nwin;       // windows
  int64_t rb;     // output blocks per destination range
  int64_t span;   // positions per destination range (rb * block)
  int nrange;     // destination ranges
  int64_t chunks_per_range;
  int64_t cells;  // nwin * nrange
  int64_t cap;    // pair slots per cell (mean + 8 sigma + 32); the rest overflow
  bool own;       // owned-run mode (k_pb_scatter_own / k_pb_reduce_own)
  int jb, bb;     // own: block = 2^jb positions, 2^bb blocks per scatter chunk
  int rthreads;   // own: reduce threads per CTA
  size_t smem;    // own: reduce shared memory
};

// window shift: 2^S entries of x per window, a window of at most `mb` MB, at least 16 windows, at most kPbMaxWin
static int pb_shift(int64_t n, int M, int64_t mb) {
  int S = 21;
  if (const char* e = getenv("NE_PB_WINDOW_MB")) mb = atoll(e);  // experiments
  while (S > 4 && (int64_t)M * 8 << S > (mb << 20)) --S;
  while (S > 4 && (n >> S) < 16) --S;
  while (((n + (1ll << S) - 1) >> S) > kPbMaxWin) ++S;
  return S;
}

static PbGeo pb_geo(int64_t n, int M, int64_t block) {
  PbGeo g{};
#ifndef NE_PB_WINDOW_MB
#define NE_PB_WINDOW_MB 32  // shared-atomic reduce (r02: best of 16-64)
#endif
#ifndef NE_PO_WINDOW_MB
#define NE_PO_WINDOW_MB 64  // owned-run reduce (r02: 64 MB 3.9-4.0 ms vs 32 MB 4.1-4.5 ms, scripts/r02/z30-z31)
#endif
  int S = pb_shift(n, M, NE_PB_WINDOW_MB);
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
  g.own = false;
  // owned-run mode: blocks that tile the scatter chunk, an index of at most
  // one entry per two positions (2 nwin <= block), a pair (j = i mod block,
  // perm[i] mod 2^S) packed in 32 bits, one reduce CTA per SM
  int jb = 0;
  while ((1ll << jb) < block) ++jb;
  S = pb_shift(n, M, NE_PO_WINDOW_MB);
  const int nwo = (int)((n + (1ll << S) - 1) >> S);
  if (block <= kPbChunk && kPbChunk % block == 0 && (1ll << jb) == block && 2 * (int64_t)nwo <= block &&
      jb + S <= 32 && (int64_t)nwo * (kPbChunk / block) <= kPbMaxWin && !kPbOwnOff && !getenv("NE_PB_NO_OWN")) {
    PbGeo o = g;
    o.own = true;
    o.S = S;
    o.nwin = nwo;
    o.jb = jb;
    o.bb = 0;
    while ((block << o.bb) < kPbChunk) ++o.bb;
    o.rb = std::max<int64_t>(1, std::min<int64_t>(kPoAccBytes / (8 * M), (nb + num_sms() - 1) / num_sms()));
    o.rb = (o.rb + 3) / 4 * 4;  // 16-byte index slices (TMA)
    o.span = o.rb * block;
    o.nrange = (int)((nb + o.rb - 1) / o.rb);
    o.chunks_per_range = (std::min<int64_t>(o.span, n) + kPbChunk - 1) / kPbChunk;
    o.cells = (int64_t)o.nwin * o.nrange;
    const int64_t mo = (n + o.cells - 1) / o.cells;
    o.cap = (mo + 8 * (int64_t)ceil(sqrt((double)mo)) + 32 + 3) / 4 * 4;
    o.rthreads = (int)std::min<int64_t>(kPoMaxThreads, ((o.rb + 1) / 2 + 31) / 32 * 32);
    o.smem = 16 + (size_t)o.rb * (M * 8 + 4) + 2 * (size_t)(o.cap + o.rb) * 4;  // k_pb_reduce_own
    if (o.cap < 65536 && o.smem <= kPoSmemMax) return o;
  }
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


#ifndef NE_PB_PREFETCH
#define NE_PB_PREFETCH 0
#endif
// TMA bulk prefetch of CTA d's share of window w of x into L2: every entry of
// a window is gathered exactly once (a permutation), so streaming the window
// in ahead of the gathers turns their DRAM misses into L2 hits
__device__ __forceinline__ void pb_prefetch_window(const int64_t* x_aos, int64_t n, int M, int S, int w, int nwin,
                                                   int d, int nparts) {
  if (!NE_PB_PREFETCH || w >= nwin) return;
  const int64_t lo = ((int64_t)w << S) * M * 8, hi = min((int64_t)(w + 1) << S, n) * M * 8;
  const int64_t share = ((hi - lo + nparts - 1) / nparts + 15) & ~15ll;
  const int64_t a = lo + (int64_t)d * share, b = min(a + share, hi) & ~15ll;
  const char* base = reinterpret_cast<const char*>(x_aos);
  for (int64_t o = a; o < b; o += 65536) {
    const uint32_t sz = (uint32_t)min((int64_t)65536, b - o);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(sz) : "memory");
  }
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
            int lockstep, int fast, int64_t n, int S, ne_streams delta) {
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
  if (threadIdx.x == 0) pb_prefetch_window(x_aos, n, M, S, 0, nwin, d, gridDim.x);
  __syncthreads();
  for (int w = 0; w < nwin; ++w) {
    if (threadIdx.x == 0) pb_prefetch_window(x_aos, n, M, S, w + 1, nwin, d, gridDim.x);
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
          asm(NE_PB_XLD " {%0,%1,%2,%3}, [%4];" : "=l"(u0), "=l"(u1), "=l"(u2), "=l"(u3) : "l"(xe));
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

// ---- owned-run mode (the C4 default when the blocks tile the chunk) ----
// The same cells, but a chunk's slice of a cell is sorted by (window, output
// block): every block's pairs in a cell form one run, and an index entry per
// (cell, block) holds the run's offset in the cell and its length (16 + 16
// bits).  A pair is packed as (i mod block) << S | (perm[i] mod 2^S) — the
// block and the window are implied by the run and the cell.  The reduce then
// needs no atomics: reduce thread t owns output blocks t, t + T, ... of its
// range and sums their runs in registers (int64 mod 2^64), window by window.
__global__ void __launch_bounds__(kPbSThreads)
k_pb_scatter_own(const int32_t* __restrict__ perm, int64_t n, int S, int nwin, int64_t span, int64_t cpr, int nrange,
                 int64_t cap, int64_t rb, int jb, int bb, unsigned* __restrict__ fill, uint32_t* __restrict__ pairs,
                 uint32_t* __restrict__ index, unsigned* __restrict__ ovn, int2* __restrict__ ov,
                 ne_diag* __restrict__ diag) {
  // block = 2^jb positions, 2^bb blocks per chunk (jb + bb = log2 kPbChunk); key = w << bb | block of the chunk
  extern __shared__ __align__(16) unsigned char smem[];
  int2* buf = reinterpret_cast<int2*>(smem);                    // [kPbChunk] (chunk-local k, perm[i]) by key
  unsigned* cnt = reinterpret_cast<unsigned*>(buf + kPbChunk);  // [kPbMaxWin]
  unsigned* off = cnt + kPbMaxWin;                              // [kPbMaxWin + 1] exclusive scan of cnt
  unsigned* gbase = off + kPbMaxWin + 1;                        // [kPbMaxWin] first slot of the window's slice
  __shared__ unsigned wsum[kPbSThreads / 32];
  int64_t c0;
  int len, d;
  pb_chunk(n, span, cpr, c0, len, d);
  const int nkey = nwin << bb;
  const int64_t blk0 = (c0 - (int64_t)d * span) >> jb;  // first block of the chunk, in its range
  for (int k = threadIdx.x; k < nkey; k += kPbSThreads) cnt[k] = 0;
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
    if (k < len && (jv[u] < 0 || jv[u] >= n)) {
      ++bad;
      first = c0 + k < first ? c0 + k : first;
      jv[u] = -1;
    }
    if (jv[u] >= 0) rk[u] = atomicAdd(&cnt[(jv[u] >> S) << bb | k >> jb], 1u);
  }
  __syncthreads();
  {  // exclusive scan over the keys: two per thread, warp scans, then the warp totals
    static_assert(2 * kPbSThreads >= kPbMaxWin, "two keys per thread");
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int k = 2 * threadIdx.x;
    const unsigned a = k < nkey ? cnt[k] : 0u, b = k + 1 < nkey ? cnt[k + 1] : 0u;
    unsigned x = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      unsigned t = lane < kPbSThreads / 32 ? wsum[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < kPbSThreads / 32) wsum[lane] = t;  // inclusive
    }
    __syncthreads();
    const unsigned ex = x - a - b + (wid ? wsum[wid - 1] : 0u);
    if (k < nkey) off[k] = ex;
    if (k + 1 < nkey) off[k + 1] = ex + a;
    if (threadIdx.x == 0) off[nkey] = wsum[kPbSThreads / 32 - 1];
  }
  __syncthreads();
  unsigned* sbase = gbase;                 // [kPbMaxWin] slot of sorted entry t of window w: sbase[w] + t (mod 2^32)
  int* lim = reinterpret_cast<int*>(buf + kPbChunk) + 3 * kPbMaxWin + 1;  // [kPbMaxWin] entries t < lim[w] fit the cell
  for (int w = threadIdx.x; w < nwin; w += kPbSThreads) {
    const unsigned sl = off[(w + 1) << bb] - off[w << bb];
    const unsigned g0 = sl ? atomicAdd(&fill[(int64_t)w * nrange + d], sl) : 0u;
    sbase[w] = (unsigned)(((uint64_t)w * nrange + d) * cap) + g0 - off[w << bb];
    lim[w] = (int)min((int64_t)off[w << bb] + cap - (int64_t)g0, (int64_t)INT_MAX);
  }
  __syncthreads();
  // the run of every (window, block of the chunk): offset in the cell, length (clipped to the capacity);
  // four blocks per 16-byte store when the chunk holds >= 4 blocks
  const int nbk = (len + (1 << jb) - 1) >> jb;
  auto run_entry = [&](int k) -> uint32_t {
    const int w = k >> bb;
    const int64_t o = (int64_t)off[k] - off[w << bb] + (cap + off[w << bb] - lim[w]);  // gbase + offset in slice
    const int64_t c = o >= cap ? 0 : min((int64_t)cnt[k], cap - o);
    return (uint32_t)min(o, cap) | (uint32_t)c << 16;
  };
  if (bb >= 2) {
    for (int k = 4 * threadIdx.x; k < nkey; k += 4 * kPbSThreads) {
      const int w = k >> bb, b = k & ((1 << bb) - 1);
      uint32_t* dst = index + ((int64_t)w * nrange + d) * rb + blk0 + b;
      if (b + 3 < nbk && blk0 + b + 3 < rb) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(run_entry(k), run_entry(k + 1), run_entry(k + 2), run_entry(k + 3));
      } else {
        for (int j = 0; j < 4; ++j)
          if (b + j < nbk && blk0 + b + j < rb) dst[j] = run_entry(k + j);
      }
    }
  } else {
    for (int k = threadIdx.x; k < nkey; k += kPbSThreads) {
      const int w = k >> bb, b = k & ((1 << bb) - 1);
      if (b >= nbk || blk0 + b >= rb) continue;
      index[((int64_t)w * nrange + d) * rb + blk0 + b] = run_entry(k);
    }
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int k = u * kPbSThreads + threadIdx.x;
    if (k < len && jv[u] >= 0) buf[off[(jv[u] >> S) << bb | k >> jb] + rk[u]] = make_int2(k, jv[u]);
  }
  __syncthreads();
  const unsigned total = off[nkey];
  const uint32_t smask = (uint32_t)((1ull << S) - 1), jmask = (1u << jb) - 1;
  for (unsigned t = threadIdx.x; t < total; t += kPbSThreads) {
    const int2 p = buf[t];
    const int w = p.y >> S;
    if ((int)t < lim[w])
      pairs[sbase[w] + t] = ((uint32_t)p.x & jmask) << S | ((uint32_t)p.y & smask);
    else
      ov[atomicAdd(ovn, 1u)] = make_int2((int32_t)(c0 + p.x), p.y);
  }
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

template <int MT>
__device__ __forceinline__ void pb_load_x(const int64_t* xe, int M, uint64_t* c) {
  if (MT == 4) {
    uint64_t u0, u1, u2, u3;
    asm(NE_PB_XLD " {%0,%1,%2,%3}, [%4];" : "=l"(u0), "=l"(u1), "=l"(u2), "=l"(u3) : "l"(xe));
    c[0] = u0; c[1] = u1; c[2] = u2; c[3] = u3;
  } else {
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : 8); ++m)
      if (MT > 0 || m < M) c[m] = (uint64_t)__ldcg(xe + m);
  }
}

// 1-D bulk copy global -> shared (TMA), completing on an mbarrier
__device__ __forceinline__ void po_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// reduce thread t owns output blocks q = t + j T (j < R per group) of its
// range; each window's cell (its pairs and its slice of the run index) is
// staged in shared memory by a 1-D TMA copy two windows ahead (double
// buffer), so a run costs only its x loads from L2; a thread's R runs are
// walked as one list (UN x loads in flight); block sums in shared memory,
// touched by their owner only
template <int MT>
__global__ void __launch_bounds__(kPoMaxThreads, 1)
k_pb_reduce_own(const int64_t* __restrict__ x_aos, int M_rt, const uint32_t* __restrict__ pairs,
                const uint32_t* __restrict__ index, const unsigned* __restrict__ fill, int64_t cap,
                unsigned* __restrict__ done, int nwin, int nrange, int64_t rb, int32_t block, int S,
                const int32_t* __restrict__ v, int32_t vlen, int64_t nb, int lockstep, int64_t n, ne_streams delta) {
  constexpr int MA = MT > 0 ? MT : 8;  // M <= 8 (host check)
#ifndef NE_PO_UN
#define NE_PO_UN 4
#endif
#ifndef NE_PO_R
#define NE_PO_R 1
#endif
  constexpr int UN = MA <= 4 ? NE_PO_UN : 2;  // x loads in flight per thread
  constexpr int R = MA <= 4 ? NE_PO_R : 2;    // runs walked together
  const int M = MT > 0 ? MT : M_rt;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);          // [2]
  uint64_t* acc = bar + 2;                                     // [rb][M]
  uint32_t* vbs = reinterpret_cast<uint32_t*>(acc + rb * M);   // [rb] (first position of block q) mod vlen
  uint32_t* stg = vbs + rb;                                     // [2][cap + rb]: pairs, then the index slice
  const int64_t stride = cap + rb;
  const int d = blockIdx.x;
  const int T = blockDim.x;
  const int64_t b0 = (int64_t)d * rb;
  const int rbl = (int)min(rb, nb - b0);
  const uint32_t smask = (uint32_t)((1ull << S) - 1);
  auto issue = [&](int w) {  // thread 0: stage window w's cell into buffer w & 1
    if (w >= nwin) return;
    const int64_t cell = (int64_t)w * nrange + d;
    const uint32_t np = (uint32_t)((min((int64_t)fill[cell], cap) + 3) & ~3ll);
    uint32_t* dst = stg + (w & 1) * stride;
    tc::mbar_expect_tx(bar + (w & 1), (np + (uint32_t)rb) * 4u);
    if (np) po_bulk_load(dst, pairs + cell * cap, np * 4u, bar + (w & 1));
    po_bulk_load(dst + cap, index + cell * rb, (uint32_t)rb * 4u, bar + (w & 1));
  };
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int q = threadIdx.x; q < rbl; q += T) {
    for (int m = 0; m < M; ++m) acc[(int64_t)q * M + m] = 0;
    vbs[q] = (uint32_t)(((b0 + q) * block) % vlen);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    issue(0);
    issue(1);
    pb_prefetch_window(x_aos, n, M, S, 0, nwin, d, gridDim.x);
  }
  for (int w = 0; w < nwin; ++w) {
    if (threadIdx.x == 0) pb_prefetch_window(x_aos, n, M, S, w + 1, nwin, d, gridDim.x);
    if (lockstep && w >= kPoLag) {  // as k_pb_reduce: at most ~3 windows of x in flight
      if (threadIdx.x == 0) {
        for (int spin = 0; spin < (1 << 20) && *(volatile unsigned*)(done + w - kPoLag) < (unsigned)nrange; ++spin)
          __nanosleep(100);
      }
      __syncthreads();
    }
    tc::mbar_wait(bar + (w & 1), (uint32_t)(w >> 1) & 1u);
    const uint32_t* pc = stg + (w & 1) * stride;
    const uint32_t* ic = pc + cap;
    const int64_t* xw = x_aos + ((int64_t)w << S) * M;
    for (int q = threadIdx.x; q < rbl; q += R * T) {
      int cum[R];
      int po[R];
      uint32_t vb[R];
      int ct = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int qj = q + j * T;
        const uint32_t e = qj < rbl ? ic[qj] : 0u;
        po[j] = (int)(e & 0xFFFFu) - ct;  // element k of run j is pc[po[j] + k]
        ct += (int)(e >> 16);
        cum[j] = ct;
        vb[j] = qj < rbl ? vbs[qj] : 0u;
      }
      uint64_t s[R][MA];
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int m = 0; m < MA; ++m) s[j][m] = 0;
      for (int k0 = 0; k0 < ct; k0 += UN) {
        uint64_t c[UN][MA];
        uint64_t wg[UN];
        int run[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int k = k0 + u;
          run[u] = R;
          if (k >= ct) continue;
          int j = 0;
#pragma unroll
          for (int jj = 0; jj < R - 1; ++jj) j += k >= cum[jj];
          run[u] = j;
          int pidx = 0;
          uint32_t vbj = 0;
#pragma unroll
          for (int jj = 0; jj < R; ++jj)
            if (jj == j) { pidx = po[jj] + k; vbj = vb[jj]; }
          const uint32_t pr = pc[pidx];
          uint32_t vi = vbj + (pr >> S);
          if (vi >= (uint32_t)vlen) vi %= (uint32_t)vlen;
          wg[u] = (uint64_t)(int64_t)__ldg(v + vi);
          pb_load_x<MT>(xw + (int64_t)(pr & smask) * M, M, c[u]);
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
#pragma unroll
          for (int m = 0; m < MA; ++m) {
            if (MT == 0 && m >= M) break;
            const uint64_t p = run[u] < R ? c[u][m] * wg[u] : 0ull;
#pragma unroll
            for (int jj = 0; jj < R; ++jj) s[jj][m] += run[u] == jj ? p : 0ull;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int qj = q + j * T;
        if (qj < rbl && cum[j] != (j ? cum[j - 1] : 0))
          for (int m = 0; m < M; ++m) acc[(int64_t)qj * M + m] += s[j][m];
      }
    }
    __syncthreads();  // buffer w & 1 consumed
    if (threadIdx.x == 0) {
      atomicAdd(done + w, 1u);
      issue(w + 2);
    }
  }
  for (int q = threadIdx.x; q < rbl; q += T)
    for (int m = 0; m < M; ++m) delta.s[m][b0 + q] = (int64_t)acc[(int64_t)q * M + m];
}

static bool pb_streams_ok(const ne_streams& c, int M) {
  for (int m = 0; m < M; ++m)
    if (!c.s[m] || !aligned16(c.s[m])) return false;
  return true;
}

}  // namespace ne

using namespace ne;

// owned-run mode: scatter (sorted runs + index), reduce (no atomics), overflow, check
static ne_status pb_run_own(const ne_config* cfg, const PbGeo& g, int M, const int64_t* x_aos, const int32_t* perm, int64_t n_total,
                            const int32_t* v, int64_t vlen, int64_t block, int64_t nb, int32_t r, ne_streams delta,
                            ne_streams d_out, uint32_t* bitmap, ne_diag* diag, void* workspace, ne_stream_t stream) {
  cudaStream_t s = cs(stream);
  uint32_t* pairs = static_cast<uint32_t*>(workspace);
  uint32_t* index = pairs + g.cells * g.cap;
  int2* ov = reinterpret_cast<int2*>(reinterpret_cast<unsigned char*>(index) +
                                     (((size_t)g.cells * g.rb * 4 + 15) & ~(size_t)15));
  unsigned* fill = reinterpret_cast<unsigned*>(ov + n_total);
  unsigned* ovn = fill + g.cells;
  unsigned* done = ovn + 1;
  if (cudaMemsetAsync(fill, 0, ((size_t)g.cells + 1 + g.nwin) * sizeof(unsigned), s) != cudaSuccess) return NE_ECUDA;
  const unsigned nchunk = (unsigned)(g.nrange * g.chunks_per_range);
  const size_t smem = (size_t)kPbChunk * sizeof(int2) + (4 * kPbMaxWin + 1) * sizeof(unsigned);
  cudaFuncSetAttribute(k_pb_scatter_own, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_pb_scatter_own<<<nchunk, kPbSThreads, smem, s>>>(perm, n_total, g.S, g.nwin, g.span, g.chunks_per_range,
                                                    g.nrange, g.cap, g.rb, g.jb, g.bb, fill, pairs, index, ovn, ov,
                                                    diag);
  const size_t rsm = g.smem;
  int per_sm = 0;
  if (cudaFuncSetAttribute(k_pb_reduce_own<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pb_reduce_own<4>, g.rthreads, rsm) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 0;
  }
  const int lockstep = g.nrange <= (int64_t)per_sm * num_sms() ? 1 : 0;
#define NE_PO_RED(MV)                                                                                            \
  cudaFuncSetAttribute(k_pb_reduce_own<MV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);              \
  k_pb_reduce_own<MV><<<g.nrange, g.rthreads, rsm, s>>>(x_aos, M, pairs, index, fill, g.cap, done, g.nwin,       \
                                                        g.nrange, g.rb, (int32_t)block, g.S, v, (int32_t)vlen,   \
                                                        nb, lockstep, n_total, delta);                           \
  k_pb_overflow<MV><<<num_sms(), 256, 0, s>>>(x_aos, M, ov, ovn, (int32_t)block, v, (int32_t)vlen, delta)
  switch (M) {
    case 4: NE_PO_RED(4); break;
    case 3: NE_PO_RED(3); break;
    case 8: NE_PO_RED(8); break;
    default: NE_PO_RED(0); break;
  }
#undef NE_PO_RED
  ne_status st = launch_status();
  if (st != NE_OK) return st;
  ne_cstreams dc{};
  for (int m = 0; m < M; ++m) dc.s[m] = delta.s[m];
  return ne_disentangle_check(cfg, dc, nb, r, d_out, bitmap, diag, stream);
}

extern "C" ne_status ne_permute_inner_workspace(const ne_config* cfg, int64_t n_total, int64_t block,
                                                size_t* bytes) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (!bytes || n_total < 0 || n_total > INT32_MAX || block < 1) return NE_EINVAL;
  const PbGeo g = pb_geo(std::max<int64_t>(n_total, 1), cfg->M, block);
  // cells at fixed capacity (owned-run mode: 32-bit pairs and the run index),
  // an overflow list as long as the input (any bijection fits), the fill
  // counters, the overflow count and the window counters
  const size_t cellb = g.own ? (size_t)g.cells * g.cap * 4 + (((size_t)g.cells * g.rb * 4 + 15) & ~(size_t)15)
                             : (size_t)g.cells * g.cap * sizeof(int2);
  *bytes = cellb + (size_t)std::max<int64_t>(n_total, 1) * sizeof(int2) +
           ((size_t)g.cells + 1 + g.nwin) * sizeof(unsigned) + 256;
  return NE_OK;
}

extern "C" ne_status ne_permute_inner_plan(const ne_config* cfg, int64_t n_total, int64_t block, int32_t* mode,
                                           int32_t* S, int32_t* nwin, int32_t* nrange, int64_t* rb, int64_t* cap,
                                           int64_t* index_bytes) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total < 0 || n_total > INT32_MAX || block < 1) return NE_EINVAL;
  const PbGeo g = pb_geo(std::max<int64_t>(n_total, 1), cfg->M, block);
  if (mode) *mode = g.own ? 1 : 0;
  if (S) *S = g.S;
  if (nwin) *nwin = g.nwin;
  if (nrange) *nrange = g.nrange;
  if (rb) *rb = g.rb;
  if (cap) *cap = g.cap;
  if (index_bytes) *index_bytes = g.own ? g.cells * g.rb * 4 : 0;
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
  if (g.own) return pb_run_own(cfg, g, M, x_aos, perm, n_total, v, vlen, block, nb, r, delta, d_out, bitmap, diag,
                               workspace, stream);
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
                                                  n_total, g.S, delta);                                                         \
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
