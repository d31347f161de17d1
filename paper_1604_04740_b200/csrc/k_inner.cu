// k_inner.cu — blocked inner product <.,.> (Eq. 2), optionally fused with the
// permutation gather (bijection I -> G) and with the disentangle +
// reliability check epilogue (Eqs. 16-19, Eq. 21) — the C4 hot path.
//
// Mapping: one warp per output block (block = 1024 positions in C4), a CTA of
// 8 warps owns 32 consecutive blocks so that it writes one whole bitmap word.
// Lane i accumulates positions i, i+32, ... in int64 (wrap mod 2^64), 8
// positions per step with all index and value loads issued before the MACs
// (memory-level parallelism for the random gather).  With the AoS layout
// (x_aos[n*M+m]) and M = 4 one gathered position is one 32-byte DRAM sector
// (2 x 128-bit loads); SoA pays one sector per stream.
#include <cuda_runtime.h>

#include <climits>

#include "ne_internal.cuh"

namespace ne {

constexpr int kBlocksPerCta = 32;
constexpr int kWarpsPerCta = 8;
constexpr int kU = 8;

template <int MT, bool AOS, bool GATHER, bool CHECK, bool VB>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
k_pinner(const __grid_constant__ ne_cstreams x, const int64_t* __restrict__ x_aos, int M_rt, int l,
         const int32_t* __restrict__ perm, int64_t n, const int32_t* __restrict__ v, int64_t vlen,
         int64_t block, const __grid_constant__ ne_streams delta_out, const __grid_constant__ ne_streams d_rot,
         int r, uint32_t* __restrict__ bitmap, ne_diag* __restrict__ diag) {
  constexpr int MA = MT > 0 ? MT : NE_MAX_M;
  const int M = MT > 0 ? MT : M_rt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nb = (n + block - 1) / block;
  __shared__ uint32_t s_flags;
  if (threadIdx.x == 0) s_flags = 0;
  __syncthreads();
  const int64_t b_first = (int64_t)blockIdx.x * kBlocksPerCta;
  int nflag = 0;
  long long first = LLONG_MAX;
  for (int bi = warp; bi < kBlocksPerCta; bi += kWarpsPerCta) {
    const int64_t b = b_first + bi;
    if (b >= nb) break;
    const int64_t p_begin = b * block;
    const int64_t p_end = p_begin + block < n ? p_begin + block : n;
    int64_t acc[MA];
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) acc[m] = 0;
    for (int64_t p0 = p_begin + lane; p0 < p_end; p0 += 32 * kU) {
      int64_t idx[kU];
      int64_t coef[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t p = p0 + 32 * u;
        const bool ok = p < p_end;
        idx[u] = ok ? (GATHER ? (int64_t)__ldcs(perm + p) : p) : -1;
        coef[u] = ok ? (int64_t)__ldg(v + (VB ? (p - p_begin) : (p % vlen))) : 0;
      }
      if (AOS && MT == 4) {
        // one 256-bit load per gathered position = exactly its 32-byte sector
        uint64_t q[kU][4];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (idx[u] >= 0) {
            asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                         : "=l"(q[u][0]), "=l"(q[u][1]), "=l"(q[u][2]), "=l"(q[u][3])
                         : "l"(x_aos + idx[u] * 4));
          } else {
            q[u][0] = q[u][1] = q[u][2] = q[u][3] = 0;
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint64_t c = (uint64_t)coef[u];
#pragma unroll
          for (int m = 0; m < 4; ++m) acc[m] = (int64_t)((uint64_t)acc[m] + q[u][m] * c);
        }
      } else {
#pragma unroll
        for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
          int64_t val[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u)
            val[u] = idx[u] >= 0 ? (AOS ? __ldcs(x_aos + idx[u] * M + m) : __ldcs(x.s[m] + idx[u])) : 0;
#pragma unroll
          for (int u = 0; u < kU; ++u) acc[m] = (int64_t)((uint64_t)acc[m] + (uint64_t)val[u] * (uint64_t)coef[u]);
        }
      }
    }
    // warp all-reduce of the M block sums
#pragma unroll
    for (int m = 0; m < (MT > 0 ? MT : M); ++m) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        acc[m] = (int64_t)((uint64_t)acc[m] + (uint64_t)__shfl_xor_sync(0xffffffffu, acc[m], o));
    }
    if (lane == 0) {
      if (delta_out.s[0]) {
#pragma unroll
        for (int m = 0; m < (MT > 0 ? MT : M); ++m) delta_out.s[m][b] = acc[m];
      }
      if (CHECK) {
        int64_t e[MA], d[MA];
        // rotated frame: e[j] = delta_{(r+j) mod M}
        if (MT > 0) {
#pragma unroll
          for (int j = 0; j < MA; ++j) {
            int src = r + j;
            if (src >= M) src -= M;
#pragma unroll
            for (int m = 0; m < MA; ++m)
              if (m == src) e[j] = acc[m];
          }
        } else {
          for (int j = 0; j < M; ++j) e[j] = acc[(r + j) % M];
        }
        const bool f = disentangle_rot<MT>(e, M, l, d, true);
#pragma unroll
        for (int j = 0; j < (MT > 0 ? MT : M); ++j) d_rot.s[j][b] = d[j];
        if (f) {
          atomicOr(&s_flags, 1u << bi);
          ++nflag;
          first = b < first ? b : first;
        }
      }
    }
  }
  if (CHECK) {
    if (diag) diag_add(&diag->fault_positions, &diag->first_fault, nflag, first);
    __syncthreads();
    if (threadIdx.x == 0 && bitmap && b_first < nb) bitmap[blockIdx.x] = s_flags;
  }
}

}  // namespace ne

using namespace ne;

template <typename S>
static bool streams_ok(const S& c, int M) {
  for (int m = 0; m < M; ++m)
    if (!c.s[m] || !aligned16(c.s[m])) return false;
  return true;
}

template <int MT, bool AOS, bool GATHER, bool CHECK>
static void launch_pinner_vb(bool vb, int grid, cudaStream_t s, const ne_cstreams& x, const int64_t* x_aos,
                             int M, int l, const int32_t* perm, int64_t n, const int32_t* v, int64_t vlen,
                             int64_t block, const ne_streams& dout, const ne_streams& drot, int r, uint32_t* bm,
                             ne_diag* diag) {
  if (vb)
    k_pinner<MT, AOS, GATHER, CHECK, true><<<grid, kWarpsPerCta * 32, 0, s>>>(x, x_aos, M, l, perm, n, v, vlen, block,
                                                                            dout, drot, r, bm, diag);
  else
    k_pinner<MT, AOS, GATHER, CHECK, false><<<grid, kWarpsPerCta * 32, 0, s>>>(x, x_aos, M, l, perm, n, v, vlen,
                                                                             block, dout, drot, r, bm, diag);
}

template <bool AOS, bool GATHER, bool CHECK>
static void launch_pinner(int M, bool vb, int grid, cudaStream_t s, const ne_cstreams& x, const int64_t* x_aos,
                          int l, const int32_t* perm, int64_t n, const int32_t* v, int64_t vlen, int64_t block,
                          const ne_streams& dout, const ne_streams& drot, int r, uint32_t* bm, ne_diag* diag) {
  switch (M) {
    case 3: launch_pinner_vb<3, AOS, GATHER, CHECK>(vb, grid, s, x, x_aos, M, l, perm, n, v, vlen, block, dout, drot, r, bm, diag); break;
    case 4: launch_pinner_vb<4, AOS, GATHER, CHECK>(vb, grid, s, x, x_aos, M, l, perm, n, v, vlen, block, dout, drot, r, bm, diag); break;
    case 8: launch_pinner_vb<8, AOS, GATHER, CHECK>(vb, grid, s, x, x_aos, M, l, perm, n, v, vlen, block, dout, drot, r, bm, diag); break;
    default: launch_pinner_vb<0, AOS, GATHER, CHECK>(vb, grid, s, x, x_aos, M, l, perm, n, v, vlen, block, dout, drot, r, bm, diag); break;
  }
}

// One stream's permutation + blocked inner product over output blocks
// [b_begin, b_begin + b_count): out_m[b - b_begin] = sum_{i in block b}
// x_m[perm[i]] v[i mod vlen] (wrap mod 2^64).  A warp per block, 8 gathers in
// flight per lane; the C4 stream-per-GPU placement.
template <bool VB>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
k_pinner_stream(const int64_t* __restrict__ x, const int32_t* __restrict__ perm, int64_t n,
                const int32_t* __restrict__ v, int64_t vlen, int64_t block, int64_t b_begin, int64_t b_count,
                int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t j = (int64_t)blockIdx.x * kWarpsPerCta + warp; j < b_count; j += (int64_t)gridDim.x * kWarpsPerCta) {
    const int64_t b = b_begin + j;
    const int64_t p_begin = b * block;
    const int64_t p_end = p_begin + block < n ? p_begin + block : n;
    uint64_t acc = 0;
    for (int64_t p0 = p_begin + lane; p0 < p_end; p0 += 32 * kU) {
      int64_t idx[kU];
      uint64_t coef[kU], val[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t p = p0 + 32 * u;
        const bool ok = p < p_end;
        idx[u] = ok ? (int64_t)__ldcs(perm + p) : -1;
        coef[u] = ok ? (uint64_t)(int64_t)__ldg(v + (VB ? (p - p_begin) : (p % vlen))) : 0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) val[u] = idx[u] >= 0 ? (uint64_t)__ldcs(x + idx[u]) : 0;
#pragma unroll
      for (int u = 0; u < kU; ++u) acc += val[u] * coef[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[j] = (int64_t)acc;
  }
}

extern "C" ne_status ne_op_permute_inner_stream(const ne_config* cfg, const int64_t* x_m, const int32_t* perm,
                                                int64_t n_total, const int32_t* v, int64_t vlen, int64_t block,
                                                int64_t b_begin, int64_t b_count, int64_t* out_m,
                                                ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total < 0 || n_total > INT32_MAX || block < 1 || vlen < 1 || !v || b_begin < 0 || b_count < 0) return NE_EINVAL;
  const int64_t nb = (n_total + block - 1) / block;
  if (b_begin + b_count > nb) return NE_EINVAL;
  if (b_count == 0) return NE_OK;
  if (!x_m || !perm || !out_m || !aligned16(x_m)) return NE_EINVAL;
  const int grid = grid_for(b_count, kWarpsPerCta, 8);
  if (vlen == block)
    k_pinner_stream<true><<<grid, kWarpsPerCta * 32, 0, cs(stream)>>>(x_m, perm, n_total, v, vlen, block, b_begin,
                                                                       b_count, out_m);
  else
    k_pinner_stream<false><<<grid, kWarpsPerCta * 32, 0, cs(stream)>>>(x_m, perm, n_total, v, vlen, block, b_begin,
                                                                        b_count, out_m);
  return launch_status();
}

extern "C" ne_status ne_op_inner(const ne_config* cfg, ne_cstreams x, int64_t n_total, const int32_t* v,
                                 int64_t vlen, int64_t block, ne_streams out, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || block < 1 || vlen < 1 || !v || !streams_ok(x, cfg->M) || !streams_ok(out, cfg->M))
    return NE_EINVAL;
  const int64_t nb = (n_total + block - 1) / block;
  const int grid = (int)((nb + kBlocksPerCta - 1) / kBlocksPerCta);
  ne_streams none{};
  launch_pinner<false, false, false>(cfg->M, vlen == block, grid, cs(stream), x, nullptr, cfg->l, nullptr, n_total,
                                     v, vlen, block, out, none, 0, nullptr, nullptr);
  return launch_status();
}

extern "C" ne_status ne_op_permute_inner_check(const ne_config* cfg, ne_cstreams x, const int64_t* x_aos,
                                               int32_t aos, const int32_t* perm, int64_t n_total,
                                               const int32_t* v, int64_t vlen, int64_t block, int32_t r,
                                               ne_streams delta_out, ne_streams d_out, uint32_t* bitmap,
                                               ne_diag* diag, ne_stream_t stream) {
  ne_status st = validate_cfg(cfg);
  if (st != NE_OK) return st;
  const int M = cfg->M;
  if (r < 0 || r >= M) return NE_EINDEX;
  if (n_total == 0) return NE_OK;
  if (n_total < 0 || n_total > INT32_MAX || block < 1 || vlen < 1 || !v || !streams_ok(d_out, M)) return NE_EINVAL;
  if (aos ? (!x_aos || !aligned16(x_aos)) : !streams_ok(x, M)) return NE_EINVAL;
  if (delta_out.s[0] && !streams_ok(delta_out, M)) return NE_EINVAL;
  const int64_t nb = (n_total + block - 1) / block;
  const int grid = (int)((nb + kBlocksPerCta - 1) / kBlocksPerCta);
  const ne_streams drot = rotate(d_out, M, r);
  const bool vb = vlen == block;
  cudaStream_t s = cs(stream);
  if (aos) {
    if (perm)
      launch_pinner<true, true, true>(M, vb, grid, s, x, x_aos, cfg->l, perm, n_total, v, vlen, block, delta_out, drot, r, bitmap, diag);
    else
      launch_pinner<true, false, true>(M, vb, grid, s, x, x_aos, cfg->l, perm, n_total, v, vlen, block, delta_out, drot, r, bitmap, diag);
  } else {
    if (perm)
      launch_pinner<false, true, true>(M, vb, grid, s, x, x_aos, cfg->l, perm, n_total, v, vlen, block, delta_out, drot, r, bitmap, diag);
    else
      launch_pinner<false, false, true>(M, vb, grid, s, x, x_aos, cfg->l, perm, n_total, v, vlen, block, delta_out, drot, r, bitmap, diag);
  }
  return launch_status();
}
