// k_gemm_pair.cu — the entangled GEMM on CTA pairs with limb-major passes
// (the C3 / C2P default for two-digit operands).  Same exact limb product as k_gemm_tc.cu (C_m = sum_i
// 2^(b i) D_{m,i} B, int8 x int8 -> int32 in TMEM, int64 recombination), with
// one 256 x 256 output tile per pair of SMs (tcgen05.mma.cta_group::2, M = 256,
// N = 256): each CTA streams its own 128 rows of A and HALF of the B columns,
// so an SM receives A + B/2 per MAC.  Each tile runs two passes over K — limb 1,
// then limb 0 — into the two halves of TMEM; the epilogue holds the finished
// limb-1 accumulators in registers and releases that half at once, so the next
// tile's limb-1 pass runs while this tile's limb 0 drains through the store
// port (the drain is hidden, as in a double-buffered kernel).  A last partial
// wave of r tiles with 2 r <= pairs runs as 2 r half tiles (256 x 128, N = 128
// MMAs; r02 A/B: the paper's M = 8, N = 2000 GEMM 81.5 -> 78.9 us, C3 280.5
// -> 280.5 us against the previous build, 282.1 with every tile whole).
//
// Pair protocol (as SM100 2-SM kernels): both CTAs' TMA loads complete on the
// LEADER's full[s] (peer bit of the barrier address cleared); the leader alone
// issues the MMAs; its commits are multicast to both CTAs' empty[s] /
// tmem_full; both CTAs' epilogue warps arrive on the leader's tmem_empty[p]
// (mapa + remote arrive).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "ne_internal.cuh"
#include "tc_common.cuh"

#ifndef NE_PAIR_STAGES  // K stages of 32 KB (6: one output staging buffer per epilogue warp; 5: two)
#define NE_PAIR_STAGES 6
#endif

namespace ne {
int gemm_max_clusters();  // ne_gemm_trace's grid cap (debug / tests), k_gemm_tc.cu
namespace tc {

// one epilogue box [32 rows x 16 int64] (or [32 x 32 int32]) to C: a TMA store
__device__ __forceinline__ void store_box(const CUtensorMap* map, int64_t c0, int64_t r0, unsigned char* box) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"((int32_t)c0), "r"((int32_t)r0), "r"(smem_u32(box))
               : "memory");
}

template <int STAGES, int SW>
struct CfgP {
  static constexpr int BN = 256;
  static constexpr int BK = SW;
  static constexpr int kATile = BM * BK;          // this CTA's 128 rows of one limb
  static constexpr int kBHalf = (BN / 2) * BK;    // this CTA's half of the B tile
  static constexpr int kStage = kATile + kBHalf;
  static constexpr int kStageOut = 32 * 16 * 8;
  static constexpr int kOutBufs = (size_t)STAGES * kStage + 2 * 8 * kStageOut + 1536 <= 232448 ? 2 : 1;
  static constexpr size_t kSmem = (size_t)STAGES * kStage + kOutBufs * 8 * kStageOut + 1024 + 256;
};

constexpr int kEpiP = 8;
constexpr int kThreadsPair = 128 + 32 * kEpiP;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the leader's copy

__device__ __forceinline__ void tma_load_pair(const CUtensorMap* map, uint64_t* bar, void* dst, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n\t"
      ".reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t"
      "}" ::"r"(smem_u32(bar))
      : "memory");
}

// L = 2: the limb-major passes above.  L = 1 (one int8 digit: the plain
// baselines, the ABFT data GEMM): one pass per tile, the two TMEM halves
// double-buffer whole tiles (tile t accumulates in half t & 1), so the drain
// of tile t overlaps the MMAs of tile t + 1.
template <int L, int STAGES, int SW, bool OUT32 = false>
__global__ void __launch_bounds__(kThreadsPair, 1)
k_gemm_pair(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
            const __grid_constant__ OutMaps outm, int64_t rows, int64_t cols, int64_t K, int M, int limb_bits,
            int raster, int64_t a_plane_rows, int toeplitz, int kcb, int64_t n_whole,
            const __grid_constant__ CUtensorMap mapBh) {
  static_assert(L == 1 || L == 2, "one or two digit planes");
  using CF = CfgP<STAGES, SW>;
  constexpr int BK = CF::BK, BN = CF::BN;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* stage_out = smem + STAGES * CF::kStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + CF::kOutBufs * 8 * CF::kStageOut);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;  // [2]: limb 1 complete, limb 0 complete
  uint64_t* tmem_empty = tmem_full + 2;  // [2]: limb-1 half, limb-0 half free (the leader's copy is used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int KB = (int)(K / BK);
  const int64_t n_rt = rows / (2 * BM), n_ct = cols / BN;
  // Work items: tiles 0 .. n_whole - 1 whole (256 x 256); the remaining tiles
  // (L = 2, the last partial wave) as two 256 x 128 halves each, item
  // n_whole + j = half j & 1 of tile n_whole + j / 2: N = 128 MMAs, half of
  // every CTA's B box (mapBh), half the epilogue chunks.  A half costs ~0.76
  // of a tile (the operand stream per MAC grows by half), so the last wave's
  // tiles spread over twice the pairs (run_pair's schedule).
  const int64_t n_tiles = (int64_t)M * n_rt * n_ct;
  const int64_t n_work = n_whole + 2 * (n_tiles - n_whole);
  const int64_t pid = blockIdx.x / 2, npair = gridDim.x / 2;
  auto decode = [&](int64_t w, int& m, int64_t& rt, int64_t& ct, int& hs) {
    int64_t t = w;
    hs = -1;
    if (w >= n_whole) {
      t = n_whole + (w - n_whole) / 2;
      hs = (int)((w - n_whole) & 1);
    }
    m = (int)(t / (n_rt * n_ct));
    const int64_t rem = t % (n_rt * n_ct);
    rt = raster ? rem % n_rt : rem / n_ct;
    ct = raster ? rem / n_rt : rem % n_ct;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full[0], 1);
    mbar_init(&tmem_full[1], 1);
    mbar_init(&tmem_empty[0], 2 * kEpiP);
    mbar_init(&tmem_empty[1], 2 * kEpiP);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
      if (n_whole < n_tiles) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBh)) : "memory");
      uint32_t it = 0;
      for (int64_t w = pid; w < n_work; w += npair) {
        int m, hs;
        int64_t rt, ct;
        decode(w, m, rt, ct, hs);
        const int64_t row0 = rt * 2 * BM + crank * BM;
        // this CTA's B rows: half of the tile's columns (a quarter of a 256-wide tile for a half item)
        const int64_t bcol0 = hs < 0 ? ct * BN + crank * (BN / 2) : ct * BN + hs * (BN / 2) + crank * (BN / 4);
        const CUtensorMap* mb = hs < 0 ? &mapB : &mapBh;
        const uint32_t tx = hs < 0 ? (uint32_t)(2 * CF::kStage) : (uint32_t)(2 * (CF::kATile + CF::kBHalf / 2));
        // K in chunks of kcb blocks, each chunk limb 1 then limb 0 (its B chunk is
        // still in L2 for the second pass); kcb = KB: one pass per limb
        for (int c0 = 0; c0 < KB; c0 += kcb)
        for (int pass = 0; pass < L; ++pass) {
          const int li = L - 1 - pass;
          for (int kb = c0; kb < KB && kb < c0 + kcb; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
            unsigned char* st = smem + s * CF::kStage;
            if (leader) mbar_expect_tx(&full[s], tx);
            // Toeplitz mode (circular conv, k_conv_tc.cu): K-chunk kb of window row b is column
            // (kb BK) mod W of row b + (kb BK) / W of the [plane_rows][W] view of the extended plane
            const int32_t kc = toeplitz ? (int32_t)(((int64_t)kb * BK) % toeplitz) : kb * BK;
            const int64_t radd = toeplitz ? ((int64_t)kb * BK) / toeplitz : 0;
            tma_load_pair(&mapA, &full[s], st, kc, (int32_t)(((int64_t)m * L + li) * a_plane_rows + row0 + radd));
            tma_load_pair(mb, &full[s], st + CF::kATile, kb * BK, (int32_t)bcol0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc_full = idesc_i8(2 * BM, BN), idesc_half = idesc_i8(2 * BM, BN / 2);
      uint32_t it = 0, tile = 0;
      for (int64_t w = pid; w < n_work; w += npair, ++tile) {
        int m, hs;
        int64_t rt, ct;
        decode(w, m, rt, ct, hs);
        const uint32_t idesc = hs < 0 ? idesc_full : idesc_half;
        for (int c0 = 0; c0 < KB; c0 += kcb)
        for (int pass = 0; pass < L; ++pass) {
          // L = 2: limb li into TMEM half li; L = 1: the tile into half tile & 1
          const int li = L == 2 ? 1 - pass : (int)(tile & 1);
          const int hb = L == 2 ? pass : li;                   // barrier pair of that half
          const uint32_t ph = L == 2 ? (tile & 1) : ((tile >> 1) & 1);
          if (c0 == 0) {
            mbar_wait(&tmem_empty[hb], ph ^ 1);  // both CTAs freed this half
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          for (int kb = c0; kb < KB && kb < c0 + kcb; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = smem_u32(smem + s * CF::kStage);
            const uint32_t sb = sa + CF::kATile;
#pragma unroll
            for (int ks = 0; ks < BK / UMMA_K; ++ks)
              mma_pair(tmem_base + li * BN, umma_desc<SW>(sa + ks * UMMA_K), umma_desc<SW>(sb + ks * UMMA_K), idesc,
                       (kb != 0 || ks != 0) ? 1u : 0u);
            commit_pair(&empty[s]);
          }
          if (c0 + kcb >= KB) commit_pair(&tmem_full[hb]);  // limb li (L = 1: the tile) complete
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = warp & 3;
    const int half = ew >> 2;
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16);
    unsigned char* my_out = stage_out + ew * CF::kOutBufs * CF::kStageOut;
    constexpr int kNch = BN / 2 / 16;
    uint32_t tile = 0, buf = 0;
    for (int64_t w = pid; w < n_work; w += npair, ++tile) {
      int m, hs;
      int64_t rt, ct;
      decode(w, m, rt, ct, hs);
      const int64_t row0 = rt * 2 * BM + crank * BM;
      // a half item (L = 2 only): columns [hs * 128, hs * 128 + 128) of the tile, 64 per warp
      const int64_t col0 = ct * BN + (hs > 0 ? BN / 2 : 0);
      const int cb = half * (hs < 0 ? BN / 2 : BN / 4);
      const int nch = hs < 0 ? kNch : kNch / 2;
      if constexpr (L == 1 && OUT32) {
        // plain int32 products (the narrowest native baseline): two 16-column TMEM
        // chunks per [32 rows x 32 int32] box, 128B swizzle, TMA store (never split)
        const int hb = (int)(tile & 1);
        mbar_wait(&tmem_full[hb], (tile >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int ci = 0; ci < kNch; ci += 2) {
          uint32_t va[16], vb[16];
          tmem_ld16(tl + hb * BN + cb + 16 * ci, va);
          tmem_ld16(tl + hb * BN + cb + 16 * (ci + 1), vb);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(va[j]), "+r"(vb[j]));
          if (ci + 2 == kNch) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) arrive_leader(&tmem_empty[hb]);
          }
          if (lane == 0) {
            if (CF::kOutBufs == 2)
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          unsigned char* box = my_out + buf * CF::kStageOut;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            *reinterpret_cast<uint4*>(box + lane * 128 + ((k ^ (lane & 7)) * 16)) =
                make_uint4(va[4 * k], va[4 * k + 1], va[4 * k + 2], va[4 * k + 3]);
            *reinterpret_cast<uint4*>(box + lane * 128 + (((k + 4) ^ (lane & 7)) * 16)) =
                make_uint4(vb[4 * k], vb[4 * k + 1], vb[4 * k + 2], vb[4 * k + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            store_box(&outm.m[m], col0 + cb + 16 * ci, row0 + 32 * q, box);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          buf = (buf + 1) % CF::kOutBufs;
        }
        continue;
      } else if constexpr (L == 1) {
        const int hb = (int)(tile & 1);
        mbar_wait(&tmem_full[hb], (tile >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t vv[2][16];
        tmem_ld16(tl + hb * BN + cb, vv[0]);
#pragma unroll
        for (int ci = 0; ci < kNch; ++ci) {
          uint32_t(&v0)[16] = vv[ci & 1];
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(v0[j]));
          if (ci + 1 < kNch) {
            tmem_ld16(tl + hb * BN + cb + 16 * (ci + 1), vv[(ci + 1) & 1]);
          } else {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) arrive_leader(&tmem_empty[hb]);
          }
          if (lane == 0) {
            if (CF::kOutBufs == 2)
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          unsigned char* box = my_out + buf * CF::kStageOut;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<longlong2*>(box + lane * 128 + ((k ^ (lane & 7)) * 16)) =
                make_longlong2((int64_t)(int32_t)v0[2 * k], (int64_t)(int32_t)v0[2 * k + 1]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            store_box(&outm.m[m], col0 + cb + 16 * ci, row0 + 32 * q, box);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          buf = (buf + 1) % CF::kOutBufs;
        }
        continue;
      }
      mbar_wait(&tmem_full[0], tile & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // hold limb 1 of this warp's columns, release that half for the next tile
      // (chunks ci >= nch are unused on a half item; indices stay compile-time)
      uint32_t hld[kNch][16];
#pragma unroll
      for (int ci = 0; ci < kNch; ++ci)
        if (ci < nch) tmem_ld16(tl + BN + cb + 16 * ci, hld[ci]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int ci = 0; ci < kNch; ++ci)
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(hld[ci][j]));
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive_leader(&tmem_empty[0]);
      mbar_wait(&tmem_full[1], tile & 1);  // limb 0 complete
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int ci = 0; ci < kNch; ++ci) {
        if (ci >= nch) break;
        const int c = cb + 16 * ci;
        uint32_t v0[16];
        tmem_ld16(tl + c, v0);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(v0[j]));
        if (ci + 1 == nch) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) arrive_leader(&tmem_empty[1]);
        }
        if (lane == 0) {
          if (CF::kOutBufs == 2)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
        unsigned char* box = my_out + buf * CF::kStageOut;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int64_t a0 = (int64_t)(int32_t)v0[2 * k] + ((int64_t)(int32_t)hld[ci][2 * k] << limb_bits);
          const int64_t a1 = (int64_t)(int32_t)v0[2 * k + 1] + ((int64_t)(int32_t)hld[ci][2 * k + 1] << limb_bits);
          *reinterpret_cast<longlong2*>(box + lane * 128 + ((k ^ (lane & 7)) * 16)) = make_longlong2(a0, a1);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          store_box(&outm.m[m], col0 + c, row0 + 32 * q, box);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        buf = (buf + 1) % CF::kOutBufs;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u));
  }
}

// Tiles kept whole by run_pair's schedule: all of them, or all but a last
// partial wave of r tiles when its 2 r halves fit one wave (2 r <= np).
// g_halves (debug hook ne_gemm_pair_halves): 0 = this rule, 1 = never halve,
// 2 = halve every tile.
static int g_halves = 0;

int64_t pair_halves(int64_t n_tiles, int64_t np) {
  if (g_halves == 1 || np < 1) return n_tiles;
  if (g_halves == 2) return 0;
  const int64_t r = n_tiles % np;
  return (r > 0 && 2 * r <= np) ? n_tiles - r : n_tiles;
}

// plain GEMM: a_plane_rows = out_rows = rows, toeplitz = 0; Toeplitz conv:
// a_plane_rows = rows of the [plane_rows][W] plane view, toeplitz = W = cols
// = 256, out_rows = output blocks (rows past it are clipped by the store)
template <int L, int STAGES, int SW, bool OUT32 = false>
static ne_status run_pair(const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, int M,
                          int limb_bits, const ne_streams& C, cudaStream_t s, int64_t a_plane_rows = 0,
                          int toeplitz = 0, int64_t out_rows = 0) {
  using CF = CfgP<STAGES, SW>;
  if (rows % (2 * BM) != 0 || cols % CF::BN != 0 || K % CF::BK != 0 || M > 8) return NE_ENOTSUP;
  if (a_plane_rows == 0) a_plane_rows = rows;
  if (out_rows == 0) out_rows = rows;
  auto kern = k_gemm_pair<L, STAGES, SW, OUT32>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::kSmem) != cudaSuccess)
    return NE_ECUDA;
  cudaLaunchConfig_t lc = {};
  lc.blockDim = dim3(kThreadsPair);
  lc.dynamicSmemBytes = CF::kSmem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  // persistent grid: one pair per two SMs, capped by how many pairs can be resident
  int64_t npairs = num_sms() / 2;
  lc.gridDim = dim3((unsigned)(npairs * 2));
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, kern, &lc) == cudaSuccess && active > 0) {
    if (active < npairs) npairs = active;
  } else {
    cudaGetLastError();
  }
  if (gemm_max_clusters() > 0 && npairs > gemm_max_clusters()) npairs = gemm_max_clusters();

  // schedule: whole 256 x 256 tiles, except (L = 2, plain GEMMs) that a last
  // partial wave of r tiles with 2 r <= pairs runs as 2 r half tiles of 256 x
  // 128 (pair_halves): a half costs ~0.76 of a tile (C3's shape with every
  // tile halved: 408.8 vs 280.7 us for twice the items); measured on the
  // tail: the paper's M = 8, N = 2000 GEMM 81.5 -> 78.9 us, C3 282.1 -> 280.5.  Split-K schedules (reduce-add into a zeroed C, or a
  // chained workspace fix-up) were measured slower: every K part
  // re-drains a whole int64 tile.
  const int64_t n_rt = rows / (2 * BM), n_ct = cols / CF::BN;
  const int64_t n_tiles = (int64_t)M * n_rt * n_ct;
  const int64_t n_whole = (L == 2 && !OUT32 && !toeplitz) ? pair_halves(n_tiles, npairs) : n_tiles;
  const int64_t n_work = n_whole + 2 * (n_tiles - n_whole);
  if (npairs > n_work) npairs = n_work;
  lc.gridDim = dim3((unsigned)(npairs * 2));
  // B panel larger than ~1/3 of L2: row tiles fastest (consecutive pairs share a B panel)
  const int raster = !toeplitz && (uint64_t)cols * (uint64_t)K > (48ull << 20) ? 1 : 0;

  CUtensorMap ma, mb, mbh;
  if (!make_map(&ma, planes, toeplitz ? (uint64_t)toeplitz : (uint64_t)K, (uint64_t)M * L * a_plane_rows, SW, BM))
    return NE_ECUDA;
  if (!make_map(&mb, Bt, (uint64_t)K, (uint64_t)cols, SW, CF::BN / 2)) return NE_ECUDA;
  if (!make_map(&mbh, Bt, (uint64_t)K, (uint64_t)cols, SW, CF::BN / 4)) return NE_ECUDA;
  OutMaps om;
  for (int m = 0; m < M; ++m) {
    if (OUT32 ? !make_out_map32(&om.m[m], C.s[m], (uint64_t)cols, (uint64_t)out_rows)
              : !make_out_map(&om.m[m], C.s[m], (uint64_t)cols, (uint64_t)out_rows))
      return NE_ECUDA;
  }
  // whole-K passes up to K = 8192 (B chunks of one pass stay in L2 at these
  // sizes); 4096-deep chunks beyond
  const int kcb = (L == 1 || K <= 8192) ? (int)(K / CF::BK) : 4096 / CF::BK;
  if (cudaLaunchKernelEx(&lc, kern, ma, mb, om, rows, cols, K, M, limb_bits, raster, a_plane_rows, toeplitz, kcb,
                         n_whole, mbh) != cudaSuccess)
    return NE_ECUDA;
  return launch_status();
}

}  // namespace tc

void gemm_pair_halves(int mode) { tc::g_halves = mode; }

int64_t gemm_pair_whole_tiles(int64_t n_tiles, int64_t npairs) { return tc::pair_halves(n_tiles, npairs); }

// Toeplitz conv with 256-output blocks and 2 limbs on the pair kernel (C2P).
ne_status launch_conv_pair(int M, int b, const int8_t* planes, int64_t plane_rows, const int8_t* Gt, int64_t Kpad,
                           int64_t nblocks, const ne_streams& C, cudaStream_t s) {
  if (b > 31 || Kpad % 128 != 0) return NE_ENOTSUP;
  const int64_t rows = (nblocks + 255) / 256 * 256;
  return tc::run_pair<2, 6, 128>(planes, Gt, rows, 256, Kpad, M, b, C, s, plane_rows, 256, nblocks);
}

// The plain (unentangled) one-digit GEMM with int32 products: the narrowest
// native baseline of the overhead comparison.  C.s[m] point to int32 buffers.
ne_status launch_gemm_pair_i32(int M, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols, int64_t K,
                               const ne_streams& C, cudaStream_t s) {
  if (K % 128 != 0) return NE_ENOTSUP;
  return tc::run_pair<1, 6, 128, true>(planes, Bt, rows, cols, K, M, 8, C, s);
}

// 256 x 256 pair tiles: 2 limbs in limb-major passes, or 1 limb with
// double-buffered tiles; NE_ENOTSUP otherwise.
ne_status launch_gemm_pair(int M, int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols,
                           int64_t K, const ne_streams& C, cudaStream_t s) {
  if (K % 128 != 0 || b > 31) return NE_ENOTSUP;
  if (L == 2) return tc::run_pair<2, NE_PAIR_STAGES, 128>(planes, Bt, rows, cols, K, M, b, C, s);
  if (L == 1) return tc::run_pair<1, NE_PAIR_STAGES, 128>(planes, Bt, rows, cols, K, M, b, C, s);
  return NE_ENOTSUP;
}

}  // namespace ne
