// k_gemm_tc2.cu — the entangled integer GEMM on CTA pairs (tcgen05
// cta_group::2): the same exact limb product as k_gemm_tc.cu (C_m =
// sum_i 2^(b i) D_{m,i} B, int8 x int8 -> int32 in TMEM, int64 recombination),
// with one 256 x BN output tile per pair of SMs of a TPC.
//
// Pair layout (rank 0 = leader, rank 1 = peer):
//   A  : each CTA loads ITS 128 rows of every limb tile (rows 128 * rank ...)
//   B  : each CTA loads HALF of the BN columns of the tile (K-major, BN/2 rows
//        of Bt); the pair's MMA reads both halves, so each SM streams half of
//        B through shared memory (the point of cta_group::2)
//   MMA: the leader alone issues tcgen05.mma.cta_group::2 (M = 256); the
//        accumulators land in both CTAs' TMEM, 128 lanes (= its rows) x L*BN
//        columns each; two accumulator sets when L * BN <= 256
//   sync: both CTAs' TMA loads complete on the LEADER's full[s] barrier (peer
//        bit cleared, as CUTLASS's SM100_TMA_2SM_LOAD), the leader's commits
//        multicast to both CTAs' empty[s] / tmem_full[b], and both CTAs'
//        epilogue warps arrive on the leader's tmem_empty[b] (mapa + remote
//        mbarrier arrive) before the leader reuses an accumulator set.
// Epilogue per CTA identical to k_gemm_tc (8 warps, tcgen05.ld 32x32b,
// 128B-swizzled int64 boxes, TMA bulk tensor stores).
#include <cuda.h>
#include <cuda_runtime.h>

#include "ne_internal.cuh"
#include "tc_common.cuh"

namespace ne {
namespace tc {

template <int L, int BN, int STAGES, int SW>
struct Cfg2 {
  static constexpr int BK = SW;
  static constexpr int kATile = BM * BK;         // this CTA's 128 rows of one limb
  static constexpr int kBHalf = (BN / 2) * BK;   // this CTA's half of the B tile
  static constexpr int kStage = L * kATile + kBHalf;
  static constexpr int kAccCols = L * BN;
  static constexpr int kBufs = 2 * kAccCols <= 512 ? 2 : 1;
  static constexpr int kNeed = kBufs * kAccCols;
  static constexpr int kTmemCols = kNeed <= 32 ? 32 : kNeed <= 64 ? 64 : kNeed <= 128 ? 128 : kNeed <= 256 ? 256 : 512;
  static constexpr int kStageOut = 32 * 16 * 8;
  static constexpr size_t kSmem = (size_t)STAGES * kStage + 2 * 8 * kStageOut + 1024 + 256;
};

constexpr int kEpiWarps2 = 8;
constexpr int kThreads2 = 128 + 32 * kEpiWarps2;
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;  // shared::cluster address of the leader's copy

__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint64_t* bar, void* dst, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
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

// arrive on the leader CTA's copy of `bar`
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n\t"
      ".reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t"
      "}" ::"r"(smem_u32(bar))
      : "memory");
}

template <int L, int BN, int STAGES, int SW>
__global__ void __launch_bounds__(kThreads2, 1)
k_gemm_tc2(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
           const __grid_constant__ OutMaps outm, int64_t rows, int64_t cols, int64_t K, int M, int limb_bits) {
  using CF = Cfg2<L, BN, STAGES, SW>;
  constexpr int BK = CF::BK;
  static_assert(L * BN <= 512 && BN % 32 == 0 && BN <= 256, "tile");
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* stage_out = smem + STAGES * CF::kStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + 2 * 8 * CF::kStageOut);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2] (the leader's copy is the one used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int KB = (int)(K / BK);
  const int64_t n_rt = rows / (2 * BM), n_ct = cols / BN;
  const int64_t n_work = (int64_t)M * n_rt * n_ct;
  const int64_t pid = blockIdx.x / 2, npair = gridDim.x / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // the leader's producer arrival (+ both CTAs' transaction bytes)
      mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 2 * kEpiWarps2);  // both CTAs' epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs: own A rows, own half of B)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
      uint32_t it = 0;
      for (int64_t w = pid; w < n_work; w += npair) {
        const int m = (int)(w / (n_rt * n_ct));
        const int64_t rem = w % (n_rt * n_ct);
        const int64_t row0 = (rem / n_ct) * 2 * BM + crank * BM;
        const int64_t bcol0 = (rem % n_ct) * BN + crank * (BN / 2);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          unsigned char* st = smem + s * CF::kStage;
          if (leader) mbar_expect_tx(&full[s], (uint32_t)(2 * CF::kStage));
#pragma unroll
          for (int i = 0; i < L; ++i)
            tma_load_2d_pair(&mapA, &full[s], st + i * CF::kATile, kb * BK,
                             (int32_t)(((int64_t)m * L + i) * rows + row0));
          tma_load_2d_pair(&mapB, &full[s], st + L * CF::kATile, kb * BK, (int32_t)bcol0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader only): M = 256 over the pair
      constexpr uint32_t idesc = idesc_i8(2 * BM, BN);
      uint32_t it = 0, tile = 0;
      for (int64_t w = pid; w < n_work; w += npair, ++tile) {
        const uint32_t ab = tile % CF::kBufs, use = tile / CF::kBufs;
        mbar_wait(&tmem_empty[ab], (use & 1) ^ 1);  // both CTAs drained this accumulator set
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * CF::kStage);
          const uint32_t sb = sa + L * CF::kATile;
#pragma unroll
          for (int ks = 0; ks < BK / UMMA_K; ++ks) {
            const uint64_t bdesc = umma_desc<SW>(sb + ks * UMMA_K);
#pragma unroll
            for (int i = 0; i < L; ++i) {
              const uint64_t adesc = umma_desc<SW>(sa + i * CF::kATile + ks * UMMA_K);
              mma_i8_pair(tmem_base + ab * CF::kAccCols + i * BN, adesc, bdesc, idesc, (kb | ks) != 0);
            }
          }
          commit_pair(&empty[s]);  // frees stage s in both CTAs
        }
        commit_pair(&tmem_full[ab]);  // this tile's accumulators are final in both CTAs
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs, own 128 rows)
    const int ew = warp - 4;
    const int q = warp & 3;
    const int half = ew >> 2;
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16);
    unsigned char* my_out = stage_out + ew * 2 * CF::kStageOut;
    uint32_t tile = 0, buf = 0;
    for (int64_t w = pid; w < n_work; w += npair, ++tile) {
      const int m = (int)(w / (n_rt * n_ct));
      const int64_t rem = w % (n_rt * n_ct);
      const int64_t row0 = (rem / n_ct) * 2 * BM + crank * BM;
      const int64_t col0 = (rem % n_ct) * BN;
      const uint32_t ab = tile % CF::kBufs, use = tile / CF::kBufs;
      mbar_wait(&tmem_full[ab], use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 16, buf ^= 1) {
        uint32_t v[L][16];
#pragma unroll
        for (int i = 0; i < L; ++i) tmem_ld16(tl + ab * CF::kAccCols + i * BN + c, v[i]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c + 16 == (half + 1) * (BN / 2)) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) arrive_leader(&tmem_empty[ab]);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        unsigned char* box = my_out + buf * CF::kStageOut;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          uint64_t a0 = 0, a1 = 0;
#pragma unroll
          for (int i = 0; i < L; ++i) {
            a0 += (uint64_t)(int64_t)(int32_t)v[i][2 * k] << (limb_bits * i);
            a1 += (uint64_t)(int64_t)(int32_t)v[i][2 * k + 1] << (limb_bits * i);
          }
          *reinterpret_cast<ulonglong2*>(box + lane * 128 + ((k ^ (lane & 7)) * 16)) = make_ulonglong2(a0, a1);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&outm.m[m])),
              "r"((int32_t)(col0 + c)), "r"((int32_t)(row0 + 32 * q)), "r"(smem_u32(box))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();  // no CTA leaves (or frees TMEM) while its peer may still use it
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)CF::kTmemCols));
  }
}

template <int L, int BN, int STAGES, int SW>
static ne_status run2(const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, int M,
                      int limb_bits, const ne_streams& C, cudaStream_t s) {
  using CF = Cfg2<L, BN, STAGES, SW>;
  if (rows % (2 * BM) != 0 || cols % BN != 0 || K % CF::BK != 0 || M > 8) return NE_ENOTSUP;
  CUtensorMap ma, mb;
  if (!make_map(&ma, planes, (uint64_t)K, (uint64_t)M * L * rows, SW, BM)) return NE_ECUDA;
  if (!make_map(&mb, Bt, (uint64_t)K, (uint64_t)cols, SW, BN / 2)) return NE_ECUDA;
  OutMaps om;
  for (int m = 0; m < M; ++m)
    if (!make_out_map(&om.m[m], C.s[m], (uint64_t)cols, (uint64_t)rows)) return NE_ECUDA;
  auto kern = k_gemm_tc2<L, BN, STAGES, SW>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::kSmem) != cudaSuccess)
    return NE_ECUDA;
  const int64_t n_work = (int64_t)M * (rows / (2 * BM)) * (cols / BN);
  cudaLaunchConfig_t lc = {};
  lc.blockDim = dim3(kThreads2);
  lc.dynamicSmemBytes = CF::kSmem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int64_t npairs = num_sms() / 2;
  lc.gridDim = dim3((unsigned)(npairs * 2));
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, kern, &lc) == cudaSuccess && active > 0) {
    if (active < npairs) npairs = active;
  } else {
    cudaGetLastError();
  }
  if (npairs > n_work) npairs = n_work;
  lc.gridDim = dim3((unsigned)(npairs * 2));
  if (cudaLaunchKernelEx(&lc, kern, ma, mb, om, rows, cols, K, M, limb_bits) != cudaSuccess) return NE_ECUDA;
  return launch_status();
}

}  // namespace tc

// CTA-pair GEMM: 256 x BN tiles; BN = 128 keeps two accumulator sets in TMEM
// for L <= 2 (the epilogue overlaps the next tile's MMAs), BN = 256 halves
// the B stream per SM further.  NE_ENOTSUP for shapes it does not tile.
ne_status launch_gemm_tc2(int M, int L, int b, int bn, const int8_t* planes, const int8_t* Bt, int64_t rows,
                          int64_t cols, int64_t K, const ne_streams& C, cudaStream_t s) {
  switch (L) {
    case 1:
      return bn == 256 ? tc::run2<1, 256, 8, 64>(planes, Bt, rows, cols, K, M, b, C, s)
                       : tc::run2<1, 128, 10, 64>(planes, Bt, rows, cols, K, M, b, C, s);
    case 2:
      return bn == 256 ? tc::run2<2, 256, 6, 64>(planes, Bt, rows, cols, K, M, b, C, s)
                       : tc::run2<2, 128, 8, 64>(planes, Bt, rows, cols, K, M, b, C, s);
    default: return NE_ENOTSUP;
  }
}

}  // namespace ne
