// k_gemm_pair.cu — the entangled GEMM on CTA pairs with limb-major passes
// (the C3 / C2P default for two-digit operands).  Same exact limb product as k_gemm_tc.cu (C_m = sum_i
// 2^(b i) D_{m,i} B, int8 x int8 -> int32 in TMEM, int64 recombination), with
// one 256 x 256 output tile per pair of SMs (tcgen05.mma.cta_group::2, M = 256,
// N = 256): each CTA streams its own 128 rows of A and HALF of the B columns,
// so an SM receives A + B/2 per MAC.  Each tile runs two passes over K — limb 1,
// then limb 0 — into the two halves of TMEM; the epilogue holds the finished
// limb-1 accumulators in registers and releases that half at once, so the next
// tile's limb-1 pass runs while this tile's limb 0 drains through the store
// port (the drain is hidden, as in a double-buffered kernel).
//
// Pair protocol (as SM100 2-SM kernels): both CTAs' TMA loads complete on the
// LEADER's full[s] (peer bit of the barrier address cleared); the leader alone
// issues the MMAs; its commits are multicast to both CTAs' empty[s] /
// tmem_full; both CTAs' epilogue warps arrive on the leader's tmem_empty[p]
// (mapa + remote arrive).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "ne_internal.cuh"
#include "tc_common.cuh"

#ifndef NE_PAIR_STAGES  // K stages of 32 KB (6: one output staging buffer per epilogue warp; 5: two)
#define NE_PAIR_STAGES 6
#endif

namespace ne {
int gemm_max_clusters();  // ne_gemm_trace's grid cap (debug / tests), k_gemm_tc.cu
namespace tc {

// one epilogue box [32 rows x 16 int64] to C: a TMA store, or a TMA
// reduce-add (u64 maps, wrap mod 2^64) when several K parts add into C
__device__ __forceinline__ void store_box(const CUtensorMap* map, int64_t c0, int64_t r0, unsigned char* box,
                                          bool add) {
  if (add)
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"((int32_t)c0), "r"((int32_t)r0), "r"(smem_u32(box))
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"((int32_t)c0), "r"((int32_t)r0), "r"(smem_u32(box))
                 : "memory");
}

#ifdef NE_PAIR_TRACE  // experiments: per CTA and item t < 32, 8 timestamps (ne_dbg_pair_trace)
__device__ long long g_pair_trace[160 * 32 * 8];
__device__ __forceinline__ void ptrace(int t, int k, long long v) {
  if (t < 32) g_pair_trace[(blockIdx.x * 32 + t) * 8 + k] = v;
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PTRACE(t, k, v) ptrace((int)(t), k, v)
#else
#define PTRACE(t, k, v)
#endif

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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
template <int L, int STAGES, int SW, bool OUT32 = false, bool SPLIT = false>
__global__ void __launch_bounds__(kThreadsPair, 1)
k_gemm_pair(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
            const __grid_constant__ OutMaps outm, int64_t rows, int64_t cols, int64_t K, int M, int limb_bits,
            int raster, int64_t a_plane_rows, int toeplitz, int kcb, int64_t n_whole, int ksplit,
            int64_t* __restrict__ ws, unsigned* __restrict__ cnt) {
  static_assert(L == 1 || L == 2, "one or two digit planes");
  static_assert(!SPLIT || (L == 2 && !OUT32), "split-K schedules: two-digit int64 tiles");
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
  // Work items: tiles 0 .. n_whole - 1 whole; the remaining n_split tiles
  // (L = 2 only) each in ksplit K parts, item n_whole + j = part j / n_split of
  // split tile ts = j mod n_split (stream-K-like fix-up: parts 0 .. ksplit - 2
  // write int64 partial tiles to the workspace ws[kp][ts][256][256] and count
  // per epilogue warp in cnt[ts][2][8]; the last part waits for its warp's
  // count, adds the partials and stores C).  Parts of a tile are ordered by w
  // and every pair takes its items in increasing w, so a waiting part only
  // waits on items already started (all pairs are resident): no deadlock.
  const int64_t n_tiles = (int64_t)M * n_rt * n_ct;
  const int64_t n_split = n_tiles - n_whole;
  const int64_t n_work = n_whole + n_split * ksplit;
  const int64_t pid = blockIdx.x / 2, npair = gridDim.x / 2;
  auto decode = [&](int64_t w, int& m, int64_t& rt, int64_t& ct, int& kb0, int& kb1, int& kp, int64_t& ts) {
    kp = 0;
    ts = -1;
    int64_t t = w;
    if (SPLIT && w >= n_whole) {
      kp = (int)((w - n_whole) / n_split);
      ts = (w - n_whole) % n_split;
      t = n_whole + ts;
    }
    const int parts = ts >= 0 ? ksplit : 1;
    m = (int)(t / (n_rt * n_ct));
    const int64_t rem = t % (n_rt * n_ct);
    rt = raster ? rem % n_rt : rem / n_ct;
    ct = raster ? rem / n_rt : rem % n_ct;
    kb0 = (int)((int64_t)kp * KB / parts);
    kb1 = (int)((int64_t)(kp + 1) * KB / parts);
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
      uint32_t it = 0;
      for (int64_t w = pid; w < n_work; w += npair) {
        int m, kb0, kb1, kp;
        int64_t rt, ct, ts;
        decode(w, m, rt, ct, kb0, kb1, kp, ts);
        const int64_t row0 = rt * 2 * BM + crank * BM;
        const int64_t bcol0 = ct * BN + crank * (BN / 2);
        // K in chunks of kcb blocks, each chunk limb 1 then limb 0 (its B chunk is
        // still in L2 for the second pass); kcb = KB: one pass per limb
        for (int c0 = kb0; c0 < kb1; c0 += kcb)
        for (int pass = 0; pass < L; ++pass) {
          const int li = L - 1 - pass;
          for (int kb = c0; kb < kb1 && kb < c0 + kcb; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
            unsigned char* st = smem + s * CF::kStage;
            if (leader) mbar_expect_tx(&full[s], (uint32_t)(2 * CF::kStage));
            // Toeplitz mode (circular conv, k_conv_tc.cu): K-chunk kb of window row b is column
            // (kb BK) mod W of row b + (kb BK) / W of the [plane_rows][W] view of the extended plane
            const int32_t kc = toeplitz ? (int32_t)(((int64_t)kb * BK) % toeplitz) : kb * BK;
            const int64_t radd = toeplitz ? ((int64_t)kb * BK) / toeplitz : 0;
            tma_load_pair(&mapA, &full[s], st, kc, (int32_t)(((int64_t)m * L + li) * a_plane_rows + row0 + radd));
            tma_load_pair(&mapB, &full[s], st + CF::kATile, kb * BK, (int32_t)bcol0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = idesc_i8(2 * BM, BN);
      uint32_t it = 0, tile = 0;
      for (int64_t w = pid; w < n_work; w += npair, ++tile) {
        int m, kb0, kb1, kp;
        int64_t rt, ct, ts;
        decode(w, m, rt, ct, kb0, kb1, kp, ts);
        for (int c0 = kb0; c0 < kb1; c0 += kcb)
        for (int pass = 0; pass < L; ++pass) {
          // L = 2: limb li into TMEM half li; L = 1: the tile into half tile & 1
          const int li = L == 2 ? 1 - pass : (int)(tile & 1);
          const int hb = L == 2 ? pass : li;                   // barrier pair of that half
          const uint32_t ph = L == 2 ? (tile & 1) : ((tile >> 1) & 1);
          if (c0 == kb0) {
            mbar_wait(&tmem_empty[hb], ph ^ 1);  // both CTAs freed this half
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            PTRACE(tile, 1 + pass, gtimer());
          }
          for (int kb = c0; kb < kb1 && kb < c0 + kcb; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = smem_u32(smem + s * CF::kStage);
            const uint32_t sb = sa + CF::kATile;
#pragma unroll
            for (int ks = 0; ks < BK / UMMA_K; ++ks)
              mma_pair(tmem_base + li * BN, umma_desc<SW>(sa + ks * UMMA_K), umma_desc<SW>(sb + ks * UMMA_K), idesc,
                       (kb != kb0 || ks != 0) ? 1u : 0u);
            commit_pair(&empty[s]);
          }
          if (c0 + kcb >= kb1) commit_pair(&tmem_full[hb]);  // limb li (L = 1: the tile) complete
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
      int m, kb0, kb1, kp;
      int64_t rt, ct, ts;
      decode(w, m, rt, ct, kb0, kb1, kp, ts);
      const int64_t row0 = rt * 2 * BM + crank * BM;
      const int64_t col0 = ct * BN;
      const int cb = half * (BN / 2);
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
            store_box(&outm.m[m], col0 + cb + 16 * ci, row0 + 32 * q, box, false);
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
            store_box(&outm.m[m], col0 + cb + 16 * ci, row0 + 32 * q, box, false);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          buf = (buf + 1) % CF::kOutBufs;
        }
        continue;
      }
      if (SPLIT && ts >= 0) {
        // a K part of a split tile (the schedule's tail: both limbs are read
        // from TMEM at the end, both halves released after the last chunk).
        // The parts form a chain: part kp waits until part kp - 1 has
        // written its running sum W_{kp-1} (this warp's box of it), adds it to
        // its own values and writes W_kp to the workspace (om.m[8], rows
        // [kp][ts][256]) — or, the last part, to C.  Own values go to the
        // smem box lane = row (as every epilogue); the previous sum is read
        // coalesced (4 rows x 128 B per warp load, one chunk ahead) and added
        // in the box piece by piece.
        const bool fin = kp == ksplit - 1;
        unsigned* wcnt = cnt + ts * 16 + crank * 8 + ew;
        const int64_t prow = crank * BM + 32 * q;   // this warp's first row in the pair tile
        // W_{kp-1}: [32 rows][256 cols] int64 slab of this warp; lane reads row lane / 8 + 4 it, piece lane % 8
        const int64_t* wprev =
            kp > 0 ? ws + (((int64_t)(kp - 1) * n_split + ts) * 256 + prow + (lane >> 3)) * 256 + cb + 2 * (lane & 7)
                   : nullptr;
        mbar_wait(&tmem_full[0], tile & 1);
        mbar_wait(&tmem_full[1], tile & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (ew == 0 && lane == 0) {
          PTRACE(tile, 0, w);
          PTRACE(tile, 3, gtimer());
        }
        longlong2 qn[8];
        if (kp > 0) {
          if (lane == 0) {
            while (ld_acquire_u32(wcnt) < (unsigned)kp) __nanosleep(32);
          }
          __syncwarp();
#pragma unroll
          for (int it = 0; it < 8; ++it) qn[it] = __ldcg(reinterpret_cast<const longlong2*>(wprev + it * 4 * 256));
        }
        if (ew == 0 && lane == 0) PTRACE(tile, 4, gtimer());
#pragma unroll 1
        for (int ci = 0; ci < kNch; ++ci) {
          const int c = cb + 16 * ci;
          uint32_t v0[16], v1[16];
          tmem_ld16(tl + BN + c, v1);
          tmem_ld16(tl + c, v0);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(v0[j]), "+r"(v1[j]));
          if (ci + 1 == kNch) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              arrive_leader(&tmem_empty[0]);
              arrive_leader(&tmem_empty[1]);
            }
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
            const int64_t a0 = (int64_t)(int32_t)v0[2 * k] + ((int64_t)(int32_t)v1[2 * k] << limb_bits);
            const int64_t a1 = (int64_t)(int32_t)v0[2 * k + 1] + ((int64_t)(int32_t)v1[2 * k + 1] << limb_bits);
            *reinterpret_cast<longlong2*>(box + lane * 128 + ((k ^ (lane & 7)) * 16)) = make_longlong2(a0, a1);
          }
          if (kp > 0) {
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int r = it * 4 + (lane >> 3), k = lane & 7;
              longlong2* pc = reinterpret_cast<longlong2*>(box + r * 128 + ((k ^ (r & 7)) * 16));
              longlong2 v = *pc;
              v.x += qn[it].x;
              v.y += qn[it].y;
              *pc = v;
            }
            if (ci + 1 < kNch)  // the next chunk's loads fly during this chunk's store
#pragma unroll
              for (int it = 0; it < 8; ++it)
                qn[it] = __ldcg(reinterpret_cast<const longlong2*>(wprev + it * 4 * 256 + 16 * (ci + 1)));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (fin)
              store_box(&outm.m[m], col0 + c, row0 + 32 * q, box, false);
            else
              store_box(&outm.m[8], c, ((int64_t)kp * n_split + ts) * 256 + prow, box, false);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          buf = (buf + 1) % CF::kOutBufs;
        }
        if (!fin && lane == 0) {  // W_kp of this warp complete in global: release it to part kp + 1
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          atomicAdd(wcnt, 1u);
        }
        if (ew == 0 && lane == 0) PTRACE(tile, 5, gtimer());
        __syncwarp();
        continue;
      }
      mbar_wait(&tmem_full[0], tile & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // hold limb 1 of this warp's columns, release that half for the next tile
      uint32_t hld[kNch][16];
#pragma unroll
      for (int ci = 0; ci < kNch; ++ci) tmem_ld16(tl + BN + cb + 16 * ci, hld[ci]);
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
      if (ew == 0 && lane == 0) {
        PTRACE(tile, 0, w);
        PTRACE(tile, 3, gtimer());
      }
#pragma unroll
      for (int ci = 0; ci < kNch; ++ci) {
        const int c = cb + 16 * ci;
        uint32_t v0[16];
        tmem_ld16(tl + c, v0);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(v0[j]));
        if (ci + 1 == kNch) {
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
          store_box(&outm.m[m], col0 + c, row0 + 32 * q, box, false);
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

// Schedule of n_tiles pair tiles over np resident pairs (static round robin):
// whole tiles only, or whole waves then the remaining tiles each in s K parts
// with the workspace fix-up.  Makespan in whole-tile units: whole waves + the
// rounds of parts, each 1/s of a tile plus an overhead f per part (pipeline
// ramp, the partial tile's write and read: about 1.5 us against 0.77 us per
// 128-deep K block of a two-pass tile, f = 2 / KB); the split is taken when it
// saves more than 3 %.  g_split forces s (debug hook ne_gemm_pair_split: 1 =
// whole tiles, s >= 2 = every tile in s parts).
static int g_split = 0;

void pair_schedule(int64_t n_tiles, int64_t np, int KB, int64_t* n_whole, int* ksplit) {
  *n_whole = n_tiles;
  *ksplit = 1;
  if (np <= 0 || n_tiles <= 0) return;
  if (g_split > 0) {
    const int sf = std::min(g_split, std::max(KB, 1));
    if (sf > 1) *n_whole = 0;
    *ksplit = sf;
    return;
  }
  const double f = 2.0 / std::max(KB, 1);
  double best = (double)((n_tiles + np - 1) / np);
  const double base = best;
  for (int64_t k = n_tiles / np; k >= 0 && k >= n_tiles / np - 2; --k) {
    const int64_t rest = n_tiles - k * np;
    if (rest <= 0) continue;
    for (int sp = 2; sp <= 8 && sp <= KB; ++sp) {
      const double mk = (double)k + (double)((rest * sp + np - 1) / np) * (1.0 / sp + f);
      if (mk < best * 0.99) {  // a larger split only for a clear gain
        best = mk;
        *n_whole = k * np;
        *ksplit = sp;
      }
    }
  }
  if (best > 0.97 * base) {
    *n_whole = n_tiles;
    *ksplit = 1;
  }
}

// the library's stream-ordered pool for split-K workspaces (one per device,
// kept warm: release threshold = max), so a launch allocates its partial
// tiles and counters on its own stream — also inside graph capture (memory
// nodes) — and concurrent launches on other streams never share them
static cudaMemPool_t split_pool() {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps pp = {};
  pp.allocType = cudaMemAllocationTypePinned;
  pp.location.type = cudaMemLocationTypeDevice;
  pp.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &pp) != cudaSuccess) {
    cudaGetLastError();
    pool = nullptr;
  } else {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  pools[dev] = pool;
  return pool;
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

  // schedule: whole tiles, or (L = 2) whole waves then the remaining tiles in
  // K parts with the workspace fix-up (pair_schedule; the workspace and the
  // counters are allocated per launch from the library's stream-ordered pool)
  const int64_t n_rt = rows / (2 * BM), n_ct = cols / CF::BN;
  const int64_t n_tiles = (int64_t)M * n_rt * n_ct;
  int64_t n_whole = n_tiles;
  int ksplit = 1;
  if (L == 2 && !OUT32) pair_schedule(n_tiles, npairs, (int)(K / CF::BK), &n_whole, &ksplit);
  cudaMemPool_t pool = ksplit > 1 ? split_pool() : nullptr;
  if (!pool) {
    n_whole = n_tiles;
    ksplit = 1;
  }
  const int64_t n_work = n_whole + (n_tiles - n_whole) * ksplit;
  if (npairs > n_work) npairs = n_work;
  lc.gridDim = dim3((unsigned)(npairs * 2));
  // B panel larger than ~1/3 of L2: row tiles fastest (consecutive pairs share a B panel)
  const int raster = !toeplitz && (uint64_t)cols * (uint64_t)K > (48ull << 20) ? 1 : 0;

  CUtensorMap ma, mb;
  if (!make_map(&ma, planes, toeplitz ? (uint64_t)toeplitz : (uint64_t)K, (uint64_t)M * L * a_plane_rows, SW, BM))
    return NE_ECUDA;
  if (!make_map(&mb, Bt, (uint64_t)K, (uint64_t)cols, SW, CF::BN / 2)) return NE_ECUDA;
  OutMaps om;
  for (int m = 0; m < M; ++m) {
    if (OUT32 ? !make_out_map32(&om.m[m], C.s[m], (uint64_t)cols, (uint64_t)out_rows)
              : !make_out_map(&om.m[m], C.s[m], (uint64_t)cols, (uint64_t)out_rows))
      return NE_ECUDA;
  }
  // whole-K passes up to K = 8192 (B chunks of one pass stay in L2 at these
  // sizes); 4096-deep chunks beyond
  const int kcb = (L == 1 || K <= 8192) ? (int)(K / CF::BK) : 4096 / CF::BK;
  cudaError_t e;
  if constexpr (L == 2 && !OUT32) {
    if (ksplit > 1) {
      // partial tiles [ksplit - 1][n_split][256][256] int64, then the counters
      const size_t n_split = (size_t)(n_tiles - n_whole);
      const size_t wsb = (size_t)(ksplit - 1) * n_split * 256 * 256 * 8;
      void* wsp = nullptr;
      if (cudaMallocFromPoolAsync(&wsp, wsb + n_split * 16 * sizeof(unsigned), pool, s) != cudaSuccess)
        return NE_ECUDA;
      int64_t* ws = static_cast<int64_t*>(wsp);
      unsigned* cnt = reinterpret_cast<unsigned*>(static_cast<char*>(wsp) + wsb);
      if (!make_out_map(&om.m[8], ws, 256, (uint64_t)(ksplit - 1) * n_split * 256) ||
          cudaMemsetAsync(cnt, 0, n_split * 16 * sizeof(unsigned), s) != cudaSuccess) {
        cudaFreeAsync(wsp, s);
        return NE_ECUDA;
      }
      auto ks = k_gemm_pair<L, STAGES, SW, false, true>;
      if (cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::kSmem) != cudaSuccess)
        return NE_ECUDA;
      e = cudaLaunchKernelEx(&lc, ks, ma, mb, om, rows, cols, K, M, limb_bits, raster, a_plane_rows, toeplitz, kcb,
                             n_whole, ksplit, ws, cnt);
      if (cudaFreeAsync(wsp, s) != cudaSuccess && e == cudaSuccess) e = cudaErrorUnknown;
    } else {
      e = cudaLaunchKernelEx(&lc, kern, ma, mb, om, rows, cols, K, M, limb_bits, raster, a_plane_rows, toeplitz,
                             kcb, n_whole, ksplit, (int64_t*)nullptr, (unsigned*)nullptr);
    }
  } else {
    e = cudaLaunchKernelEx(&lc, kern, ma, mb, om, rows, cols, K, M, limb_bits, raster, a_plane_rows, toeplitz, kcb,
                           n_whole, ksplit, (int64_t*)nullptr, (unsigned*)nullptr);
  }
  if (e != cudaSuccess) return NE_ECUDA;
  return launch_status();
}

}  // namespace tc

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

void gemm_pair_split(int s) { tc::g_split = s; }

#ifdef NE_PAIR_TRACE
extern "C" int ne_dbg_pair_trace(long long* host, int reset) {
  if (reset) {
    static long long zero[160 * 32 * 8];
    return cudaMemcpyToSymbol(tc::g_pair_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : 1;
  }
  return cudaMemcpyFromSymbol(host, tc::g_pair_trace, sizeof(long long) * 160 * 32 * 8) == cudaSuccess ? 0 : 1;
}
#endif

void gemm_pair_schedule(int64_t n_tiles, int64_t npairs, int KB, int64_t* n_whole, int* ksplit) {
  tc::pair_schedule(n_tiles, npairs, KB, n_whole, ksplit);
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
