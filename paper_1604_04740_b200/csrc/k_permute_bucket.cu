// k_permute_bucket.cu — the fused permutation + blocked inner product of C4 as
// a partitioned scatter-reduce: no random DRAM gather, no global atomics on
// the sums.
//
// The op (P:253-258 permutation, then the blocked inner product of Eq. 2):
//   delta_m[b] = sum_{i in block b} x_m[perm[i]] * v[i mod vlen]
// The gather form (k_inner.cu, k_pinner) reads x at random positions: every
// 32-byte AoS entry costs a 128-byte DRAM line fill (profiles/r02_c4_floor.md).
// Here the pairs (i, perm[i]) are partitioned into cells (w, d): w = the
// source window perm[i] >> S (2^S entries of x, a slice of L2), d = the
// destination range of RB output blocks that i falls in (RB x M int64 sums
// fit one CTA's shared memory).  Cells are laid out window-major.
//   pass 1 (k_pb_count): per chunk of consecutive i (one d per chunk), a
//     shared-memory histogram over w, one atomic per (chunk, w) into the cell
//     counts;
//   pass 2 (k_pb_scan): exclusive scan of the counts (window-major) -> cell
//     offsets;
//   pass 3 (k_pb_scatter): per chunk again, the pairs sorted by w in shared
//     memory and written to their cells (one atomic per (chunk, w) reserves
//     the slice), window-grouped;
//   pass 4 (k_pb_reduce): CTA d walks its cells w = 0, 1, ... in window order
//     (all CTAs move through x window by window, so the window being read is
//     in L2), gathers x[perm[i]] from L2, and adds the M products with
//     v[i mod vlen] into its shared-memory block sums (pairs of 32-bit shared
//     atomics with carry; a soft lockstep keeps the CTAs within two windows);
//     it then writes its RB blocks of delta once (no global atomics);
//   then ne_disentangle_check on delta, exactly as the gather path.
// Every sum is an int64 sum mod 2^64, so delta is bit-identical to the gather
// order (wrap-free for certified results).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "ne_internal.cuh"

namespace ne {

constexpr int kPbChunk = 8192;      // positions per count / scatter CTA (one destination range)
constexpr int kPbThreads = 512;
constexpr int kPbMaxWin = 1024;     // windows
constexpr int kPbAccBytes = 32768;  // shared block sums per reduce CTA

struct PbGeo {
  int S;          // window shift
  int nwin;       // windows
  int64_t rb;     // output blocks per destination range
  int64_t span;   // positions per destination range (rb * block)
  int nrange;     // destination ranges
  int64_t chunks_per_range;
  int64_t cells;  // nwin * nrange
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

__global__ void __launch_bounds__(kPbThreads)
k_pb_count(const int32_t* __restrict__ perm, int64_t n, int S, int nwin, int64_t span, int64_t cpr, int nrange,
           unsigned* __restrict__ count, ne_diag* __restrict__ diag) {
  __shared__ unsigned h[kPbMaxWin];
  int64_t c0;
  int len, d;
  pb_chunk(n, span, cpr, c0, len, d);
  for (int w = threadIdx.x; w < nwin; w += kPbThreads) h[w] = 0;
  __syncthreads();
  int bad = 0;
  long long first = LLONG_MAX;
  for (int k = threadIdx.x; k < len; k += kPbThreads) {
    const int32_t j = __ldcs(perm + c0 + k);
    if (j < 0 || j >= n) {  // not a permutation of [0, n): counted here, skipped by every pass
      ++bad;
      first = c0 + k < first ? c0 + k : first;
    } else {
      atomicAdd(&h[j >> S], 1u);
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < nwin; w += kPbThreads)
    if (h[w]) atomicAdd(&count[(int64_t)w * nrange + d], h[w]);
  if (diag) diag_add(&diag->range_violations, &diag->first_bad, bad, first);
}

// exclusive scan of the cell counts -> offsets (one CTA of 1024 threads)
__global__ void __launch_bounds__(1024) k_pb_scan(const unsigned* __restrict__ count, int64_t cells,
                                                  unsigned* __restrict__ offset) {
  __shared__ unsigned part[1024];
  const int64_t per = (cells + 1023) / 1024;
  const int64_t lo = min(threadIdx.x * per, cells), hi = min(lo + per, cells);
  unsigned s = 0;
  for (int64_t k = lo; k < hi; ++k) s += count[k];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // inclusive Hillis-Steele scan of the partials
    const unsigned t = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  unsigned acc = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  for (int64_t k = lo; k < hi; ++k) {
    offset[k] = acc;
    acc += count[k];
  }
}

__global__ void __launch_bounds__(kPbThreads)
k_pb_scatter(const int32_t* __restrict__ perm, int64_t n, int S, int nwin, int64_t span, int64_t cpr, int nrange,
             const unsigned* __restrict__ offset, unsigned* __restrict__ fill, int2* __restrict__ pairs) {
  extern __shared__ __align__(16) unsigned char smem[];
  int2* buf = reinterpret_cast<int2*>(smem);                    // [kPbChunk]
  unsigned* cnt = reinterpret_cast<unsigned*>(buf + kPbChunk);  // [kPbMaxWin]
  unsigned* off = cnt + kPbMaxWin;                              // [kPbMaxWin] chunk-local offsets
  unsigned* gbase = off + kPbMaxWin;                            // [kPbMaxWin] first slot in the cell
  int64_t c0;
  int len, d;
  pb_chunk(n, span, cpr, c0, len, d);
  for (int w = threadIdx.x; w < nwin; w += kPbThreads) cnt[w] = 0;
  __syncthreads();
  constexpr int kPer = kPbChunk / kPbThreads;
  int32_t jv[kPer];
  unsigned rk[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int k = u * kPbThreads + threadIdx.x;
    jv[u] = k < len ? __ldcs(perm + c0 + k) : -1;
    if (jv[u] >= n) jv[u] = -1;
    if (jv[u] >= 0) rk[u] = atomicAdd(&cnt[jv[u] >> S], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // chunk-local exclusive scan over windows
    unsigned acc = 0;
    for (int w = 0; w < nwin; ++w) {
      off[w] = acc;
      acc += cnt[w];
    }
  }
  for (int w = threadIdx.x; w < nwin; w += kPbThreads) {
    const int64_t cell = (int64_t)w * nrange + d;
    gbase[w] = cnt[w] ? offset[cell] + atomicAdd(&fill[cell], cnt[w]) : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int k = u * kPbThreads + threadIdx.x;
    if (k < len && jv[u] >= 0) buf[off[jv[u] >> S] + rk[u]] = make_int2((int32_t)(c0 + k), jv[u]);
  }
  __syncthreads();
  const unsigned total = off[nwin - 1] + cnt[nwin - 1];
  for (unsigned k = threadIdx.x; k < total; k += kPbThreads) {
    const int2 p = buf[k];
    const int w = p.y >> S;
    pairs[gbase[w] + (k - off[w])] = p;
  }
}

template <int MT>
__global__ void __launch_bounds__(kPbThreads)
k_pb_reduce(const int64_t* __restrict__ x_aos, int M_rt, const int2* __restrict__ pairs,
            const unsigned* __restrict__ count, const unsigned* __restrict__ offset, unsigned* __restrict__ done,
            int nwin, int nrange, int64_t rb, int32_t block, const int32_t* __restrict__ v, int32_t vlen, int64_t nb,
            int lockstep, ne_streams delta) {
  constexpr int MA = MT > 0 ? MT : 8;  // M <= 8 (host check)
  const int M = MT > 0 ? MT : M_rt;
  // block sums as (low, high) 32-bit words: two native 32-bit shared atomics
  // per add (a 64-bit shared atomicAdd is a CAS loop on this target), the
  // carry out of the low word added to the high word by the add that caused
  // it — exact mod 2^64
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
      if (threadIdx.x == 0)
        while (*(volatile unsigned*)(done + w - 2) < (unsigned)nrange) __nanosleep(100);
      __syncthreads();
    }
    const int64_t cell = (int64_t)w * nrange + d;
    const unsigned lo = offset[cell], cnt = count[cell];
    for (unsigned k = threadIdx.x; k < cnt; k += kPbThreads) {
      const int2 pr = __ldcs(pairs + lo + k);
      const uint64_t wgt = (uint64_t)(int64_t)__ldg(v + pr.x % vlen);
      const int bl = (int)(pr.x / block - b0);
      const int64_t* xe = x_aos + (int64_t)pr.y * M;
      uint64_t c[MA];
      if (MT == 4) {
        uint64_t u0, u1, u2, u3;
        asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(u0), "=l"(u1), "=l"(u2), "=l"(u3) : "l"(xe));
        c[0] = u0; c[1] = u1; c[2] = u2; c[3] = u3;
      } else {
#pragma unroll
        for (int m = 0; m < (MT > 0 ? MT : M); ++m) c[m] = (uint64_t)__ldg(xe + m);
      }
#pragma unroll
      for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
        const uint64_t p = c[m] * wgt;
        unsigned* a = acc + 2 * (bl * M + m);
        const unsigned lo = (unsigned)p, old = atomicAdd(a, lo);
        atomicAdd(a + 1, (unsigned)(p >> 32) + (old + lo < old ? 1u : 0u));
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
    delta.s[m][b0 + bl] = (int64_t)(((uint64_t)acc[2 * k + 1] << 32) | acc[2 * k]);
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
  *bytes = (size_t)std::max<int64_t>(n_total, 1) * sizeof(int2) + ((size_t)g.cells * 3 + g.nwin) * sizeof(unsigned) +
           256;
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
  unsigned* count = reinterpret_cast<unsigned*>(pairs + n_total);
  unsigned* offset = count + g.cells;
  unsigned* fill = offset + g.cells;
  unsigned* done = fill + g.cells;
  if (cudaMemsetAsync(count, 0, (size_t)g.cells * sizeof(unsigned), s) != cudaSuccess ||
      cudaMemsetAsync(fill, 0, ((size_t)g.cells + g.nwin) * sizeof(unsigned), s) != cudaSuccess)
    return NE_ECUDA;
  const unsigned nchunk = (unsigned)(g.nrange * g.chunks_per_range);
  k_pb_count<<<nchunk, kPbThreads, 0, s>>>(perm, n_total, g.S, g.nwin, g.span, g.chunks_per_range, g.nrange, count,
                                           diag);
  k_pb_scan<<<1, 1024, 0, s>>>(count, g.cells, offset);
  const size_t smem = (size_t)kPbChunk * sizeof(int2) + 3 * kPbMaxWin * sizeof(unsigned);
  cudaFuncSetAttribute(k_pb_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_pb_scatter<<<nchunk, kPbThreads, smem, s>>>(perm, n_total, g.S, g.nwin, g.span, g.chunks_per_range, g.nrange,
                                                offset, fill, pairs);
  // the window lockstep needs every reduce CTA resident at once
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pb_reduce<4>, kPbThreads, 0) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 0;
  }
  const int lockstep = g.nrange <= (int64_t)per_sm * num_sms() ? 1 : 0;
#define NE_PB_RED(MV)                                                                                             \
  k_pb_reduce<MV><<<g.nrange, kPbThreads, 0, s>>>(x_aos, M, pairs, count, offset, done, g.nwin, g.nrange, g.rb,   \
                                                  (int32_t)block, v, (int32_t)vlen, nb, lockstep, delta)
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
