// k_gemm_tc.cu — the entangled integer GEMM on the 5th-generation tensor
// cores (tcgen05.mma kind::i8), exact.
//
// C_m = E_m B with E_m the entangled rows x K operand (Eq. 9) and
// B the shared K x cols kernel (unmodified).  E_m is held as L balanced signed
// base-2^8 digit planes D_{m,i} (ne_entangle_limbs / k_split_limbs), B as one
// int8 plane (|B| <= 128), so
//     C_m = sum_i 2^(8i) (D_{m,i} B),
// every D_{m,i} B is an int8 x int8 -> int32 tensor-core product that is exact
// while K * 128 * 128 < 2^31 (K < 131072), and the recombination is done in
// int64 in the epilogue (wrap mod 2^64, exact for certified results).  The
// digit base 2^b is a launch parameter: b = 8 (any operand) or b = l (an
// entangled operand c_m + 2^l c_{m-1} whose halves fit int8: 2 limbs).
//
// A CTA computes 128 x BN tiles of one stream at a time: the L limb
// accumulators live side by side in TMEM (L * BN <= 512 columns).  Roles:
//   warp 0 lane 0 : TMA producer  (cp.async.bulk.tensor, 64B or 128B swizzle, multicast, mbarrier complete_tx)
//   warp 1 lane 0 : MMA issuer    (tcgen05.mma.cta_group::1.kind::i8, commit -> mbarrier)
//   warp 2        : TMEM allocator (tcgen05.alloc / dealloc)
//   warps 4..11   : epilogue      (tcgen05.ld 32x32b -> int64 recombine -> swizzled smem -> TMA store);
//                   warp w reads TMEM lane quarter w%4, column half (w-4)/4; the TMEM load of
//                   the next 16-column chunk is in flight while the current one is staged
//   warps 12..19  : checkers (CHK > 0 only: the fused disentangle + check)
// smem: STAGES x {L limb tiles 128 x BK, one B tile BN x BK} (BK = 64 or 128 bytes of K,
// swizzle of the same width), 1024-B aligned; clusters of 2 CTAs along N multicast
// the limb tiles (or along M the B tile, Toeplitz mode).  Output modes: one
// tensor map per stream, or per destination row block (Geo::dest_rows, the C5
// fused exchange).  DESIGN.md §7 has the measured per-tile timeline: with one
// TMEM accumulator set (L * BN = 512) the ~4.5 us drain of each 256 KB int64
// tile through the SM's store port is not overlapped.
#include <cuda.h>
#include <cuda_runtime.h>

#include "ne_internal.cuh"
#include "tc_common.cuh"

namespace ne {
namespace tc {

template <int L, int BN, int STAGES, int SW, int CL>
struct Cfg {
  static constexpr int BK = SW;                   // bytes (= int8 elements) of K per stage
  static constexpr int kATile = BM * BK;          // one limb tile
  static constexpr int kBTile = BN * BK;
  static constexpr int kStage = L * kATile + kBTile;
  static constexpr int kARows = BM / CL;          // rows of each limb tile this CTA loads (multicast)
  static constexpr int kAccCols = L * BN;                     // one accumulator set
  static constexpr int kBufs = 2 * kAccCols <= 512 ? 2 : 1;   // double-buffered when two sets fit TMEM
  static constexpr int kTmemNeed = kBufs * kAccCols;
  static constexpr int kTmemCols = (kTmemNeed <= 32) ? 32 : (kTmemNeed <= 64) ? 64 : (kTmemNeed <= 128) ? 128 : (kTmemNeed <= 256) ? 256 : 512;
  static constexpr int kStageOut = 32 * 16 * 8;  // one epilogue warp's [32 rows x 16 int64] box
  // staging boxes per epilogue warp: 2 (double-buffered TMA stores) unless the
  // operand stages leave room for only 1 in the 227 KB of shared memory
  static constexpr int kOutBufs = (size_t)STAGES * kStage + 2 * 8 * kStageOut + 1536 <= 232448 ? 2 : 1;
  static constexpr size_t kSmem = (size_t)STAGES * kStage + kOutBufs * 8 * kStageOut + 1024 /*align*/ + 512 /*barriers, check queue*/;
};


// Fused a4/a5 (CHK = M > 0): the M streams' tiles of one output tile are
// consecutive work items (stream index fastest), so they run at about the
// same time on M different CTAs.  Each CTA, once its delta tile is stored
// (bulk stores complete, proxy fence, release), increments the tile's counter.
// Tile t is checked by the CTA computing stream t mod M (balanced): its
// epilogue queues t for the CTA's 8 checker warps, which wait until the
// counter reaches M, read the M delta tiles back and run disentangle + check
// (Eqs. 16-19, 21), writing d_hat, the bitmap and ne_diag exactly as
// k_disentangle<M, true> does, then re-zero the counter.  The checkers never
// touch TMEM, so the MMA pipeline does not wait for them.  The delta tiles are
// the op's stored outputs: the check still sees every stream through memory.
// Measured: correct, but slower than GEMM + separate check on
// B200 — the checker warps' 800 MB of extra memory traffic per C3 step is
// latency-bound at 8 warps per SM and stretches the GEMM by ~0.16 ms.
struct ChkArgs {
  ne_cstreams dr;     // delta, rotated so that the excluded stream r is index 0
  ne_streams dor;     // d_hat outputs, same rotation
  uint32_t* bitmap;   // nullable
  ne_diag* diag;      // nullable
  int* cnt;           // (rows/128) x (cols/BN) zero-initialised tile counters
  int l;
};

// Operand geometry.  GEMM: A is the [M*L*rows][K] stack of limb planes and C_m
// is [rows][cols].  Toeplitz (circular convolution as a GEMM, k_conv_tc.cu;
// toeplitz = the output block width W in {128, 256}): each limb plane is a
// circularly extended 1-D stream of a_plane_rows * W bytes viewed as
// [a_plane_rows][W]; window row b of K bytes starts at byte W b, so the K-chunk
// kb (BK bytes) of row b is column (kb BK) mod W of row b + (kb BK) / W of
// that view (no overlapping tensor-map strides needed).  Output rows >=
// out_rows are clipped by the TMA store (tensor bounds).
// mcast_b (clusters of CL > 1): the CL CTAs of a cluster take CL consecutive
// row tiles of the same column tile and share the B tile instead of the A
// tile (each loads BN/CL rows of B and multicasts them) — the convolution's
// G matrix is shared by every work item, its A windows by none.
// raster_rows: row tiles fastest in the work order (consecutive clusters
// share a column group of B instead of a row tile of A) — chosen when B does
// not fit L2 next to the A operand, so each B panel is read from DRAM ~once.
// dest_rows (> 0, a multiple of 128; GEMM with M = 1 only): output row block
// j = row / dest_rows goes to out map j, at row - j * dest_rows — the fused
// GEMM -> position-major exchange of C5, each map addressing the owner rank's
// receive buffer (peer memory over NVLink, or local); with dest_local the
// tile is also stored at its own row through out map 8 (the full local copy
// that recovery after a fail-stop needs).
struct Geo {
  int64_t a_plane_rows;
  int64_t out_rows;
  int toeplitz;  // 0, or the Toeplitz output block width W in bytes (= outputs)
  int mcast_b;
  int raster_rows;
  int64_t dest_rows;
  int dest_local;
};

// Digit plan of one launch (ne_op_gemm_planes; the default is the plain
// L-digit base-2^b product): accumulator i holds A plane a0 + i (of a_total
// planes per stream) times the B plane whose rows start at b_row0 of the
// [LB * cols][K] B-plane stack, and carries bit weight sh[i] in the int64
// recombination.  accumulate: the epilogue adds its tile into C with a TMA
// reduce-add (u64, wrap mod 2^64) instead of storing it — the later launches
// of a multi-launch plan (more than 4 A planes, or several B planes).
struct Plan {
  int sh[4];
  int small;      // every sh[i] <= 30: 32 x 32 -> 64-bit multiply-adds
  int a_total;
  int a0;
  int64_t b_row0;
  int accumulate;
};

__host__ __device__ inline Plan plain_plan(int L, int b) {
  Plan p{};
  for (int i = 0; i < 4; ++i) p.sh[i] = i < L ? b * i : 0;
  p.small = b * (L - 1) <= 30;
  p.a_total = L;
  return p;
}

// Debug hook (ne_gemm_trace): per CTA and tile t < 32, %globaltimer when the
// tile's accumulators are complete and when its last chunk is staged.
struct DbgArgs {
  long long* trace;
};
__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
static long long* g_trace = nullptr;
static int g_max_clusters = 0;

__device__ __forceinline__ void epi_bar() {  // the 8 epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(32 * 8) : "memory");
}

constexpr int kChkWarps = 8;  // checker warps (fused check only; 4 and 16 measured slower)
constexpr int kChkThreads = 32 * kChkWarps;

__device__ __forceinline__ void chk_bar() {  // the checker warps only
  asm volatile("bar.sync 2, %0;" ::"n"(kChkThreads) : "memory");
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// spread the low 16 bits of x to the even bit positions (bitmap assembly)
__device__ __forceinline__ uint32_t spread16e(uint32_t x) {
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// disentangle + check of one 128 x BN output tile by the checker threads
// (et = 0..kChkThreads-1): pair p = j*kChkThreads + et covers row p / (BN/2), columns
// col0 + 2 (p % (BN/2)) .. +1, so a warp owns 64 consecutive positions of a
// row = two bitmap words (as in k_disentangle).  Loads go through L2 (.cg:
// the tiles were written by this kernel), U pairs in flight per thread.
template <int MT, int BN>
__device__ __forceinline__ void check_tile(const ChkArgs& chk, int64_t row0, int64_t col0, int64_t cols,
                                           int64_t n_total, int et) {
  constexpr int U = MT >= 4 ? 2 : 4;  // registers: <= 96 per thread at 640 threads
  constexpr int kPairs = BM * BN / 2;
  static_assert(kPairs % (kChkThreads * U) == 0, "tile pairs divide evenly");
  const int lane = et & 31;
  int nflag = 0;
  long long first = LLONG_MAX;
#pragma unroll 1
  for (int j0 = 0; j0 < kPairs / kChkThreads; j0 += U) {
    int64_t a[U][MT], b[U][MT], n0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int p = (j0 + u) * kChkThreads + et;
      n0[u] = (row0 + p / (BN / 2)) * cols + col0 + 2 * (p % (BN / 2));
#pragma unroll
      for (int s = 0; s < MT; ++s) {
        const longlong2 q = __ldcg(reinterpret_cast<const longlong2*>(chk.dr.s[s] + n0[u]));
        a[u][s] = q.x;
        b[u][s] = q.y;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t da[MT], db[MT];
      const bool f0 = disentangle_rot<MT>(a[u], MT, chk.l, da, true);
      const bool f1 = disentangle_rot<MT>(b[u], MT, chk.l, db, true);
#pragma unroll
      for (int s = 0; s < MT; ++s)
        __stcs(reinterpret_cast<longlong2*>(chk.dor.s[s] + n0[u]), make_longlong2(da[s], db[s]));
      if (f0) {
        ++nflag;
        first = n0[u] < first ? n0[u] : first;
      }
      if (f1) {
        ++nflag;
        first = n0[u] + 1 < first ? n0[u] + 1 : first;
      }
      if (chk.bitmap) {
        const uint32_t b0 = __ballot_sync(0xffffffffu, f0);
        const uint32_t b1 = __ballot_sync(0xffffffffu, f1);
        const int64_t w0 = (n0[u] - 2 * lane) / 32;  // lane 0's position starts a 64-position run
        if (lane == 0) chk.bitmap[w0] = spread16e(b0) | (spread16e(b1) << 1);
        if (lane == 1) chk.bitmap[w0 + 1] = spread16e(b0 >> 16) | (spread16e(b1 >> 16) << 1);
      }
    }
  }
  (void)n_total;
  if (chk.diag) diag_add(&chk.diag->fault_positions, &chk.diag->first_fault, nflag, first);
}

// Persistent, warp-specialised kernel.  The grid is one CTA per SM (clusters
// of CL along N); each cluster walks the work list w = cid, cid + nclusters, ...
// with w -> (stream m, row tile, column-tile group), CTA rank r taking column
// tile group*CL + r.  The CL CTAs of a cluster share the row tile: each loads
// 128/CL rows of every limb tile and multicasts them to all CL CTAs, so A is
// read from L2 once per cluster.  Accumulators: two sets of L * BN TMEM
// columns when they fit (L * BN <= 256: the MMA of tile t+1 runs while the
// epilogue drains tile t), else one set (L * BN = 512): the MMA warp waits
// until the epilogue has drained TMEM (tmem_empty) before the next tile,
// while the producer already streams the next tile's stages; the epilogue's
// global stores drain under the next mainloop.
constexpr int kEpiWarps = 8;
constexpr int kThreadsP = 128 + 32 * kEpiWarps;  // warps 0-3: roles, 4-11: epilogue
template <int CHK>
constexpr int threads_for() { return kThreadsP + (CHK > 0 ? 32 * kChkWarps : 0); }
constexpr int kQN = 32;                          // check queue ring (tile ids)

// work item w -> (stream m, row tile, column-tile group); stream-fastest
// order when the check is fused (CHK > 0), else stream-slowest
template <int CHK>
__device__ __forceinline__ void decode_work(int64_t w, int M, int64_t n_rt, int64_t n_cg, int& m, int64_t& rt,
                                            int64_t& cg, int raster_rows) {
  if (CHK == 0 && raster_rows) {
    m = (int)(w / (n_rt * n_cg));
    const int64_t rem = w % (n_rt * n_cg);
    cg = rem / n_rt;
    rt = rem % n_rt;
  } else if (CHK > 0) {
    m = (int)(w % M);
    const int64_t rem = w / M;
    rt = rem / n_cg;
    cg = rem % n_cg;
  } else {
    m = (int)(w / (n_rt * n_cg));
    const int64_t rem = w % (n_rt * n_cg);
    rt = rem / n_cg;
    cg = rem % n_cg;
  }
}

template <int L, int BN, int STAGES, int SW, int CL, int CHK>
__global__ void __launch_bounds__(threads_for<CHK>(), 1)
k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
          const __grid_constant__ OutMaps outm, int64_t rows, int64_t cols, int64_t K, int M,
          const __grid_constant__ ChkArgs chk, const Geo geo, const DbgArgs dbg, const Plan pl) {
  using CF = Cfg<L, BN, STAGES, SW, CL>;
  constexpr int BK = CF::BK;
  static_assert(L * BN <= 512, "TMEM holds 512 columns");
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* stage_out = smem + STAGES * CF::kStage;  // 2 x 8 x 4 KB, 1024-B aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + CF::kOutBufs * 8 * CF::kStageOut);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;  // [kBufs]
  uint64_t* tmem_empty = tmem_full + 2;  // [kBufs]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  // check queue (CHK > 0): ring of tile ids pushed by the epilogue, consumed by the checker warps
  volatile int* q_head = reinterpret_cast<volatile int*>(tmem_slot + 1);
  volatile int* q_tail = q_head + 1;
  volatile int* q_done = q_head + 2;
  volatile int* q_ring = q_head + 4;
  if (threadIdx.x == 0) {
    *q_head = 0;
    *q_tail = 0;
    *q_done = 0;
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = CL > 1 ? cluster_rank() : 0;
  const uint16_t cmask = (uint16_t)((1u << CL) - 1);
  const int KB = (int)(K / BK);
  const bool mb = CL > 1 && geo.mcast_b;
  const int64_t n_rt = mb ? rows / (BM * CL) : rows / BM, n_cg = mb ? cols / BN : cols / (BN * CL);
  const int64_t n_work = (int64_t)M * n_rt * n_cg;
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // released by the MMA warp of every CTA in the cluster
    }
    for (int b = 0; b < CF::kBufs; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CL > 1)
    cluster_sync();  // peers' barriers are initialised before anyone multicasts
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
      uint32_t it = 0;
      for (int64_t w = cid; w < n_work; w += ncl) {
        int m;
        int64_t rt, cg;
        decode_work<CHK>(w, M, n_rt, n_cg, m, rt, cg, geo.raster_rows);
        const int64_t row0 = mb ? (rt * CL + crank) * BM : rt * BM;
        const int64_t col0 = mb ? cg * BN : (cg * CL + crank) * BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          unsigned char* st = smem + s * CF::kStage;
          mbar_expect_tx(&full[s], (uint32_t)CF::kStage);
          const int32_t kc = geo.toeplitz ? (int32_t)(((int64_t)kb * BK) % geo.toeplitz) : kb * BK;
          const int64_t radd = geo.toeplitz ? ((int64_t)kb * BK) / geo.toeplitz : 0;
          if (mb) {
#pragma unroll
            for (int i = 0; i < L; ++i) {
              const int32_t grow =
                  (int32_t)(((int64_t)m * pl.a_total + pl.a0 + i) * geo.a_plane_rows + row0 + radd);
              tma_load_2d(&mapA, &full[s], st + i * CF::kATile, kc, grow);
            }
            tma_load_2d_mc(&mapB, &full[s], st + L * CF::kATile + crank * (BN / CL) * BK, kb * BK,
                           (int32_t)(pl.b_row0 + col0 + crank * (BN / CL)), cmask);
          } else {
#pragma unroll
            for (int i = 0; i < L; ++i) {
              unsigned char* dst = st + i * CF::kATile + crank * CF::kARows * BK;
              const int32_t grow = (int32_t)(((int64_t)m * pl.a_total + pl.a0 + i) * geo.a_plane_rows + row0 +
                                             crank * CF::kARows + radd);
              if (CL > 1)
                tma_load_2d_mc(&mapA, &full[s], dst, kc, grow, cmask);
              else
                tma_load_2d(&mapA, &full[s], dst, kc, grow);
            }
            tma_load_2d(&mapB, &full[s], st + L * CF::kATile, kb * BK, (int32_t)(pl.b_row0 + col0));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_i8(BM, BN);
      uint32_t it = 0, tile = 0;
      for (int64_t w = cid; w < n_work; w += ncl, ++tile) {
        const uint32_t ab = tile % CF::kBufs, use = tile / CF::kBufs;
        mbar_wait(&tmem_empty[ab], (use & 1) ^ 1);  // epilogue drained this accumulator set
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        long long t_wait = 0;
        if (dbg.trace && tile < 32) dbg.trace[(blockIdx.x * 32 + tile) * 4 + 2] = globaltimer();
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          if (dbg.trace) {
            const long long t0 = globaltimer();
            mbar_wait(&full[s], (it / STAGES) & 1);
            t_wait += globaltimer() - t0;
          } else {
            mbar_wait(&full[s], (it / STAGES) & 1);
          }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * CF::kStage);
          const uint32_t sb = sa + L * CF::kATile;
#pragma unroll
          for (int ks = 0; ks < BK / UMMA_K; ++ks) {
            const uint64_t bdesc = umma_desc<SW>(sb + ks * UMMA_K);
#pragma unroll
            for (int i = 0; i < L; ++i) {
              const uint64_t adesc = umma_desc<SW>(sa + i * CF::kATile + ks * UMMA_K);
              mma_i8(tmem_base + ab * CF::kAccCols + i * BN, adesc, bdesc, idesc, (kb | ks) != 0);
            }
          }
          mma_commit(&empty[s], cmask);  // frees stage s in every CTA of the cluster
        }
        mma_commit(&tmem_full[ab], 1);   // this tile's accumulators are final
        if (dbg.trace && tile < 32) dbg.trace[(blockIdx.x * 32 + tile) * 4 + 3] = t_wait;
      }
    }
  } else if (warp >= 4 && warp < 4 + kEpiWarps) {
    // ---------------- epilogue: TMEM -> registers -> int64 recombination ->
    // 128B-swizzled smem box -> TMA bulk tensor store (double-buffered per warp)
    const int ew = warp - 4;
    const int q = warp & 3;          // TMEM lane quarter this warp may access (warp id mod 4)
    const int half = ew >> 2;        // column half
    const uint32_t tl = tmem_base + ((uint32_t)(32 * q) << 16);
    unsigned char* my_out = stage_out + ew * CF::kOutBufs * CF::kStageOut;
    uint32_t tile = 0, buf = 0;
    for (int64_t w = cid; w < n_work; w += ncl, ++tile) {
      int m;
      int64_t rt, cg;
      decode_work<CHK>(w, M, n_rt, n_cg, m, rt, cg, geo.raster_rows);
      const int64_t row0 = mb ? (rt * CL + crank) * BM : rt * BM;
      const int64_t col0 = mb ? cg * BN : (cg * CL + crank) * BN;
      const uint32_t ab = tile % CF::kBufs, use = tile / CF::kBufs;
      mbar_wait(&tmem_full[ab], use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (dbg.trace && ew == 0 && lane == 0 && tile < 32) dbg.trace[(blockIdx.x * 32 + tile) * 4] = globaltimer();
      // 16-column chunks, kNch per warp; the TMEM load of chunk ci+1 is in
      // flight while chunk ci is staged (two register sets, plain GEMM only)
      constexpr int kNch = BN / 2 / 16;
      constexpr bool kPipe = CHK == 0 && L <= 3;  // (L = 4: 128 registers of limbs would spill)
      const uint32_t tacc = tl + ab * CF::kAccCols;
      const int cb = half * (BN / 2);
      uint32_t vs[kPipe ? 2 : 1][L][16];
      // stage one chunk: pack the limbs to int64, 128B-swizzled smem box, TMA store
      auto stage = [&](uint32_t(&v)[L][16], int c) {
        // the TMA store that last read this buffer must be done
        if (lane == 0) {
          if (CF::kOutBufs == 2)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
        unsigned char* box = my_out + buf * CF::kStageOut;
        // row `lane` of the box, 16-byte chunk k stored at chunk k ^ (row & 7) (128B swizzle)
        if (pl.small) {  // sum_i v_i 2^sh_i as 32 x 32 -> 64-bit multiply-adds
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            int64_t a0 = (int64_t)(int32_t)v[0][2 * k] * (1 << pl.sh[0]);
            int64_t a1 = (int64_t)(int32_t)v[0][2 * k + 1] * (1 << pl.sh[0]);
#pragma unroll
            for (int i = 1; i < L; ++i) {
              const int32_t sc = 1 << pl.sh[i];
              a0 += (int64_t)(int32_t)v[i][2 * k] * sc;
              a1 += (int64_t)(int32_t)v[i][2 * k + 1] * sc;
            }
            *reinterpret_cast<longlong2*>(box + lane * 128 + ((k ^ (lane & 7)) * 16)) = make_longlong2(a0, a1);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            uint64_t a0 = 0, a1 = 0;
#pragma unroll
            for (int i = 0; i < L; ++i) {
              a0 += (uint64_t)(int64_t)(int32_t)v[i][2 * k] << pl.sh[i];
              a1 += (uint64_t)(int64_t)(int32_t)v[i][2 * k + 1] << pl.sh[i];
            }
            *reinterpret_cast<ulonglong2*>(box + lane * 128 + ((k ^ (lane & 7)) * 16)) = make_ulonglong2(a0, a1);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const int dj = geo.dest_rows > 0 ? (int)(row0 / geo.dest_rows) : m;  // destination map
          const int64_t drow = geo.dest_rows > 0 ? row0 - dj * geo.dest_rows : row0;
          if (pl.accumulate)  // C += tile (u64 maps: wrap mod 2^64, exact for certified sums)
            asm volatile(
                "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&outm.m[dj])),
                "r"((int32_t)(col0 + c)), "r"((int32_t)(drow + 32 * q)), "r"(smem_u32(box))
                : "memory");
          else
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&outm.m[dj])),
              "r"((int32_t)(col0 + c)), "r"((int32_t)(drow + 32 * q)), "r"(smem_u32(box))
              : "memory");
          if (geo.dest_local)
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&outm.m[8])),
                "r"((int32_t)(col0 + c)), "r"((int32_t)(row0 + 32 * q)), "r"(smem_u32(box))
                : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        buf = (buf + 1) % CF::kOutBufs;
      };
#pragma unroll
      for (int i = 0; i < L; ++i) tmem_ld16(tacc + i * BN + cb, vs[0][i]);
#pragma unroll
      for (int ci = 0; ci < kNch; ++ci) {
        uint32_t(&v)[L][16] = vs[kPipe ? (ci & 1) : 0];
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < L; ++i)
#pragma unroll
          for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(v[i][j]));  // uses stay after the wait
        if (kPipe && ci + 1 < kNch) {
#pragma unroll
          for (int i = 0; i < L; ++i) tmem_ld16(tacc + i * BN + cb + 16 * (ci + 1), vs[(ci + 1) & 1][i]);
        }
        if (ci + 1 == kNch) {
          // last TMEM read of this tile for this warp: release the accumulators
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[ab])) : "memory");
        }
        stage(v, cb + 16 * ci);
        if (!kPipe && ci + 1 < kNch) {
#pragma unroll
          for (int i = 0; i < L; ++i) tmem_ld16(tacc + i * BN + cb + 16 * (ci + 1), vs[0][i]);
        }
      }
      if (dbg.trace && ew == 0 && lane == 0 && tile < 32) dbg.trace[(blockIdx.x * 32 + tile) * 4 + 1] = globaltimer();
      if constexpr (CHK > 0) {
        // publish this delta tile: bulk stores complete and ordered before
        // the generic-proxy reads of the CTA that checks the tile
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __syncwarp();
        epi_bar();
        const int64_t tile_id = rt * (cols / BN) + cg * CL + crank;
        if (ew == 0 && lane == 0) {
          __threadfence();
          atomicAdd(chk.cnt + tile_id, 1);
          if (tile_id % M == m) {  // this CTA's checker warps check the tile (balanced: 1 in M)
            const int h = *q_head;
            while (h - *q_tail >= kQN) __nanosleep(128);
            q_ring[h % kQN] = (int)tile_id;
            __threadfence_block();
            *q_head = h + 1;
          }
        }
      }
    }
    if constexpr (CHK > 0) {
      if (ew == 0 && lane == 0) {
        __threadfence_block();
        *q_done = 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp >= 4 + kEpiWarps) {
    if constexpr (CHK > 0) {
    // ---------------- checkers: disentangle + check of the tiles queued for
    // this CTA, once all M streams' delta tiles are published (tile counter == M)
    const int ct = threadIdx.x - 32 * (4 + kEpiWarps);  // 0 .. kChkThreads-1
    int tail = 0;
    while (true) {
      const int done = *q_done;
      const int head = *q_head;
      if (tail == head) {
        if (done) break;
        __nanosleep(256);
        continue;
      }
      __threadfence_block();
      const int tile_id = q_ring[tail % kQN];
      if (ct == 0) {
        // bounded wait (all CTAs are co-resident: the grid is sized by the
        // cluster occupancy); a timeout is reported as a flagged run, not a hang
        long long spins = 0;
        int c;
        while ((c = ld_acquire(chk.cnt + tile_id)) < M && ++spins < (1ll << 24)) __nanosleep(64);
        if (c < M && chk.diag) atomicAdd(&chk.diag->fault_positions, 1ull << 40);
      }
      chk_bar();
      const int64_t nct = cols / BN;
      check_tile<CHK, BN>(chk, (tile_id / nct) * BM, (tile_id % nct) * BN, cols, rows * cols, ct);
      chk_bar();
      ++tail;
      if (ct == 0) {
        chk.cnt[tile_id] = 0;
        *q_tail = tail;
      }
    }
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CL > 1)
    cluster_sync();  // no CTA leaves while a peer may still signal its barriers
  else
    __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)CF::kTmemCols));
  }
}

// ---------------------------------------------------------------- host side
template <int L, int BN, int STAGES, int SW, int CL, int CHK = 0>
static ne_status run(const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, int M,
                     int limb_bits, const ne_streams& C, cudaStream_t s, const ChkArgs* chk = nullptr,
                     const Geo* geo_in = nullptr, const Plan* plan_in = nullptr, int LB = 1) {
  using CF = Cfg<L, BN, STAGES, SW, CL>;
  const Plan pl = plan_in ? *plan_in : plain_plan(L, limb_bits);
  if (cols % BN != 0 || K % CF::BK != 0) return NE_ENOTSUP;
  // B panel larger than ~1/3 of L2: rasterise along rows (see Geo)
  const int raster = (CHK == 0 && (uint64_t)cols * (uint64_t)K > (48ull << 20)) ? 1 : 0;
  const Geo geo = geo_in ? *geo_in : Geo{rows, rows, 0, 0, raster};
  const bool mcb = CL > 1 && geo.mcast_b;
  if (mcb && rows % (BM * CL) != 0) return NE_ENOTSUP;
  if (!mcb && cols % (BN * CL) != 0) return NE_ENOTSUP;
  CUtensorMap ma, mb;
  if (!make_map(&ma, planes, geo.toeplitz ? (uint64_t)geo.toeplitz : (uint64_t)K,
                (uint64_t)M * pl.a_total * geo.a_plane_rows, SW, mcb ? BM : CF::kARows))
    return NE_ECUDA;
  if (!make_map(&mb, Bt, (uint64_t)K, (uint64_t)cols * LB, SW, mcb ? BN / CL : BN)) return NE_ECUDA;
  if (M > 8) return NE_ENOTSUP;
  OutMaps om;
  if (geo.dest_rows > 0) {  // C.s[j]: destination j's [dest_rows][cols] block
    if (M != 1 || geo.dest_rows % BM != 0 || rows % geo.dest_rows != 0 || rows / geo.dest_rows > 8)
      return NE_ENOTSUP;
    for (int j = 0; j < rows / geo.dest_rows; ++j)
      if (!make_out_map(&om.m[j], C.s[j], (uint64_t)cols, (uint64_t)geo.dest_rows)) return NE_ECUDA;
    if (geo.dest_local && !make_out_map(&om.m[8], C.s[8], (uint64_t)cols, (uint64_t)rows)) return NE_ECUDA;
  } else {
    for (int m = 0; m < M; ++m)
      if (!make_out_map(&om.m[m], C.s[m], (uint64_t)cols, (uint64_t)geo.out_rows, pl.accumulate != 0))
        return NE_ECUDA;
  }
  auto kern = k_gemm_tc<L, BN, STAGES, SW, CL, CHK>;
  ChkArgs ca{};
  if (CHK > 0) ca = *chk;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::kSmem) != cudaSuccess)
    return NE_ECUDA;
  const int64_t n_work = (int64_t)M * (rows / BM) * (cols / BN) / CL;
  cudaLaunchConfig_t lc = {};
  lc.blockDim = dim3(threads_for<CHK>());
  lc.dynamicSmemBytes = CF::kSmem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  // persistent grid: one CTA per SM, capped by how many clusters can be
  // resident at once (the fused check waits on peer CTAs' tiles, so every
  // CTA of the grid must be co-resident)
  int64_t nclusters = num_sms() / CL;
  lc.gridDim = dim3((unsigned)(nclusters * CL));
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, kern, &lc) == cudaSuccess && active > 0) {
    if (active < nclusters) nclusters = active;
  } else {
    cudaGetLastError();
    if (CHK > 0) return NE_ENOTSUP;
  }
  if (nclusters > n_work) nclusters = n_work;
  if (g_max_clusters > 0 && nclusters > g_max_clusters) nclusters = g_max_clusters;
  lc.gridDim = dim3((unsigned)(nclusters * CL));
  const DbgArgs dbg{g_trace};
  if (cudaLaunchKernelEx(&lc, kern, ma, mb, om, rows, cols, K, M, ca, geo, dbg, pl) != cudaSuccess)
    return NE_ECUDA;
  return launch_status();
}

}  // namespace tc

// Tile choice: L limb accumulators of BN columns fill TMEM (L * BN <= 512);
// 64-byte K stages (64B swizzle) give 4-6 pipeline stages in ~200 KB of smem;
// clusters of 2 along N multicast the limb tiles (A read once per pair)
// whenever the column-tile count is even.
template <int CHK>
static ne_status gemm_tc_dispatch(int M, int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows,
                                  int64_t cols, int64_t K, const ne_streams& C, cudaStream_t s, const tc::ChkArgs* chk,
                                  const tc::Geo* geo = nullptr) {
  const bool pair128 = cols % 256 == 0, pair256 = cols % 512 == 0;
  switch (L) {
    case 1:
      if (CHK > 0) return NE_ENOTSUP;
      if (pair256) return tc::run<1, 256, 6, 64, 2>(planes, Bt, rows, cols, K, M, b, C, s, nullptr, geo);
      if (cols % 256 == 0) return tc::run<1, 256, 6, 64, 1>(planes, Bt, rows, cols, K, M, b, C, s, nullptr, geo);
      return tc::run<1, 128, 8, 64, 1>(planes, Bt, rows, cols, K, M, b, C, s, nullptr, geo);
    case 2:
      // 128-byte K stages (128B swizzle, 3 stages, single-buffered store
      // staging): half the TMA row requests and barrier round trips per MAC
      // of the 64-byte / 5-stage form (C3 GEMM 0.2897 -> 0.2862 ms)
      // (long work lists only: with few waves the shallower pipeline's ramp
      // shows — the ABFT checksum GEMM, 3.5 waves, measured 5 % slower)
      if (CHK == 0 && pair256 && K % 128 == 0 && (int64_t)M * (rows / 128) * (cols / 512) >= 6 * (num_sms() / 2))
        return tc::run<2, 256, 3, 128, 2>(planes, Bt, rows, cols, K, M, b, C, s, chk, geo);
      if (pair256) return tc::run<2, 256, 5, 64, 2, CHK>(planes, Bt, rows, cols, K, M, b, C, s, chk, geo);
      if (cols % 256 == 0) return tc::run<2, 256, 5, 64, 1, CHK>(planes, Bt, rows, cols, K, M, b, C, s, chk, geo);
      return tc::run<2, 128, 6, 64, 1, CHK>(planes, Bt, rows, cols, K, M, b, C, s, chk, geo);
    case 3:
      if (CHK > 0) return NE_ENOTSUP;
      if (pair128) return tc::run<3, 128, 5, 64, 2>(planes, Bt, rows, cols, K, M, b, C, s, nullptr, geo);
      return tc::run<3, 128, 5, 64, 1>(planes, Bt, rows, cols, K, M, b, C, s, nullptr, geo);
    case 4:
      if (CHK > 0) return NE_ENOTSUP;  // 4 limb accumulators leave no registers for checker warps
      if (pair128) return tc::run<4, 128, 4, 64, 2>(planes, Bt, rows, cols, K, M, b, C, s, nullptr, geo);
      return tc::run<4, 128, 4, 64, 1>(planes, Bt, rows, cols, K, M, b, C, s, nullptr, geo);
    default: return NE_ENOTSUP;
  }
}

void gemm_trace(long long* buf, int max_clusters) {
  tc::g_trace = buf;
  tc::g_max_clusters = max_clusters;
}

int gemm_max_clusters() { return tc::g_max_clusters; }

ne_status launch_gemm_pair(int M, int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols,
                           int64_t K, const ne_streams& C, cudaStream_t s);

// The CTA-pair gate of launch_gemm_tc (also answered by ne_gemm_kernel_for).
bool gemm_pair_gate(int M, int L, int b, int64_t rows, int64_t cols, int64_t K) {
  const int64_t pair_tiles = (int64_t)M * (rows / 256) * (cols / 256);
  if (K % 128 != 0 || rows % 256 != 0 || cols % 256 != 0 || M > 8 || b > 31) return false;
  // one digit (plain baselines, ABFT data): double-buffered 256 x 256 pair
  // tiles, each SM receiving A + B/2 per MAC (the single-CTA L = 1 tile needs
  // A + B and is bound by the SM's inbound operand rate)
  if (L == 1) return K >= 1024 && pair_tiles >= 64;
#ifndef NE_PAIR_KMIN   // experiments (scripts/r02/ab.py): the smallest K the two-digit pair kernel takes
#define NE_PAIR_KMIN 2048
#define NE_PAIR_TILES_SHORTK 256
#endif
  return L == 2 && (K >= 4096 || (K >= NE_PAIR_KMIN && pair_tiles >= NE_PAIR_TILES_SHORTK)) && K <= 8192;
}

ne_status launch_gemm_tc(int M, int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols,
                         int64_t K, const ne_streams& C, cudaStream_t s) {
  // Two digits, mid-length K: the CTA-pair kernel with limb-major passes
  // (k_gemm_pair.cu) hides the int64 drain behind the next tile's first pass
  // (C3 GEMM 0.293 -> 0.277 ms).  Measured slower for short K (the paper's
  // N = 200 / 2000 shapes: the per-pass fill costs more than the drain) and for
  // C5's K = 16384 (the drain is ~6 % of a tile there), so those keep the
  // single-CTA kernel.  The debug trace hook covers the single-CTA kernel only.
  // (K = 2048 pays only with several waves of pair tiles: the paper's M = 8,
  // N = 2000 shape 0.086 -> 0.082 ms, M = 3 0.039 -> 0.041 ms; K <= 1024 never)
  if (gemm_pair_gate(M, L, b, rows, cols, K) && tc::g_trace == nullptr) {
    const ne_status st = launch_gemm_pair(M, L, b, planes, Bt, rows, cols, K, C, s);
    if (st != NE_ENOTSUP) return st;
  }
  return gemm_tc_dispatch<0>(M, L, b, planes, Bt, rows, cols, K, C, s, nullptr);
}

// One launch of a general digit plan: Lsub <= 4 A planes (accumulators) x
// one B plane, tile shapes as gemm_tc_dispatch.
static ne_status run_plan(int M, int Lsub, const int8_t* planes, const int8_t* Bt, int LB, int64_t rows,
                          int64_t cols, int64_t K, const ne_streams& C, cudaStream_t s, const tc::Plan& pl) {
  const bool c512 = cols % 512 == 0, c256 = cols % 256 == 0;
  switch (Lsub) {
    case 1:
      if (c512) return tc::run<1, 256, 6, 64, 2>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
      if (c256) return tc::run<1, 256, 6, 64, 1>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
      return tc::run<1, 128, 8, 64, 1>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
    case 2:
      if (c512) return tc::run<2, 256, 5, 64, 2>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
      if (c256) return tc::run<2, 256, 5, 64, 1>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
      return tc::run<2, 128, 6, 64, 1>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
    case 3:
      if (c256) return tc::run<3, 128, 5, 64, 2>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
      return tc::run<3, 128, 5, 64, 1>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
    case 4:
      if (c256) return tc::run<4, 128, 4, 64, 2>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
      return tc::run<4, 128, 4, 64, 1>(planes, Bt, rows, cols, K, M, 8, C, s, nullptr, nullptr, &pl, LB);
    default: return NE_ENOTSUP;
  }
}

// The general exact product C_m = sum_{i<LA} sum_{j<LB} 2^(a_shift[i] + 8 j)
// (D_{m,i} B_j): A planes in groups of <= 4 accumulators, one launch per
// (group, B plane); the first launch stores C, the others add into it (TMA
// reduce-add, wrap mod 2^64, exact for certified results).  A plain
// L <= 4 base-2^b plan with one B plane takes launch_gemm_tc (incl. the
// CTA-pair kernel).
ne_status launch_gemm_planes(int M, const int8_t* planes, int LA, const int32_t* a_shift, const int8_t* Bt, int LB,
                             int64_t rows, int64_t cols, int64_t K, const ne_streams& C, cudaStream_t s) {
  if (LA < 1 || LA > 8 || LB < 1 || LB > 5) return NE_EINVAL;
  bool uniform = LA <= 4 && LB == 1;
  const int b = LA > 1 ? a_shift[1] - a_shift[0] : 8;
  for (int i = 0; i < LA && uniform; ++i) uniform = a_shift[i] == b * i;
  if (uniform && b >= 8 && b <= 63) return launch_gemm_tc(M, LA, b, planes, Bt, rows, cols, K, C, s);
  bool first = true;
  for (int i = 0; i < LA; ++i)
    if (a_shift[i] < 0 || a_shift[i] > 63) return NE_EINVAL;
  for (int j = 0; j < LB; ++j)
    for (int g = 0; g < LA; g += 4) {
      tc::Plan pl{};
      // products of bit weight >= 64 vanish mod 2^64 (the results wrap there):
      // an accumulator group starting beyond that is skipped
      if (a_shift[g] + 8 * j >= 64) continue;
      int Lsub = LA - g < 4 ? LA - g : 4;
      while (a_shift[g + Lsub - 1] + 8 * j >= 64) --Lsub;
      int mx = 0;
      for (int i = 0; i < Lsub; ++i) {
        pl.sh[i] = a_shift[g + i] + 8 * j;
        mx = pl.sh[i] > mx ? pl.sh[i] : mx;
      }
      pl.small = mx <= 30;
      pl.a_total = LA;
      pl.a0 = g;
      pl.b_row0 = (int64_t)j * cols;
      pl.accumulate = first ? 0 : 1;
      const ne_status st = run_plan(M, Lsub, planes, Bt, LB, rows, cols, K, C, s, pl);
      if (st != NE_OK) return st;
      first = false;
    }
  return NE_OK;
}

// One stream's GEMM (M = 1) with row block j of the output stored to dests[j]
// ([rows / ndest][cols] int64 each), and in full to `local` if non-null: the
// fused GEMM -> exchange of C5.
ne_status launch_gemm_tc_scatter(int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols,
                                 int64_t K, const ne_streams& dests, int ndest, int64_t* local, cudaStream_t s) {
  const int raster = (uint64_t)cols * (uint64_t)K > (48ull << 20) ? 1 : 0;
  const tc::Geo geo{rows, rows, 0, 0, raster, rows / ndest, local ? 1 : 0};
  ne_streams d = dests;  // ne_streams holds NE_MAX_M >= 9 pointers
  d.s[8] = local;
  return gemm_tc_dispatch<0>(1, L, b, planes, Bt, rows, cols, K, d, s, nullptr, &geo);
}

// Circular convolution / correlation of M entangled streams as a Toeplitz
// GEMM (k_conv_tc.cu): planes = M*L extended limb planes of plane_rows * W
// bytes; Gt = [W][Kpad] int8 tap matrix; C_m = [nblocks][W] int64 (the first
// W * nblocks outputs of stream m).  One W-output column tile.
//   W = 128: clusters of 2 consecutive row tiles multicast the shared tap
//     tiles of G; 128-byte K stages (128B swizzle): each window row is one
//     full 128-byte line of the extended plane per stage; double-buffered
//     TMEM (L * 128 <= 256)
//   W = 256 (L <= 2): the C3 GEMM configuration (128 x 256 tiles, 64-byte K
//     stages, 5 stages) — the A windows are reused by 256 columns instead of
//     128, halving the A stream per MAC
ne_status launch_conv_pair(int M, int b, const int8_t* planes, int64_t plane_rows, const int8_t* Gt, int64_t Kpad,
                           int64_t nblocks, const ne_streams& C, cudaStream_t s);

ne_status launch_conv_tc(int M, int L, int b, int W, const int8_t* planes, int64_t plane_rows, const int8_t* Gt,
                         int64_t Kpad, int64_t nblocks, const ne_streams& C, cudaStream_t s) {
  // long kernels (1024 <= Kpad <= 8192) with 256-output blocks and two
  // digits: the CTA-pair limb-major kernel (C2P M = 8, T = 4500: conv 0.080 ->
  // 0.072 ms; T = 1000: 35.9 -> 35.0 us); at T = 300 slower (pipeline fill
  // per pass); longer kernels keep the single-CTA kernel
#ifndef NE_CONV_PAIR_KMIN  // (r02 A/B, C2P M = 8, T = 1000 at Kpad = 1280: pair 35.0 vs single-CTA 35.9 us)
#define NE_CONV_PAIR_KMIN 1024
#endif
  if (W == 256 && L == 2 && Kpad >= NE_CONV_PAIR_KMIN && Kpad <= 8192 && tc::g_trace == nullptr) {
    const ne_status st = launch_conv_pair(M, b, planes, plane_rows, Gt, Kpad, nblocks, C, s);
    if (st != NE_ENOTSUP) return st;
  }
  const tc::Geo geo{plane_rows, nblocks, W, 1, 0};
  const int64_t rows = (nblocks + 255) / 256 * 256;
  if (Kpad % 128 != 0) return NE_EINVAL;
  if (W == 256) {
    switch (L) {
      case 1: return tc::run<1, 256, 6, 64, 2>(planes, Gt, rows, 256, Kpad, M, b, C, s, nullptr, &geo);
      case 2: return tc::run<2, 256, 5, 64, 2>(planes, Gt, rows, 256, Kpad, M, b, C, s, nullptr, &geo);
      default: return NE_ENOTSUP;
    }
  }
  switch (L) {
    case 1: return tc::run<1, 128, 5, 128, 2>(planes, Gt, rows, 128, Kpad, M, b, C, s, nullptr, &geo);
    case 2: return tc::run<2, 128, 3, 128, 2>(planes, Gt, rows, 128, Kpad, M, b, C, s, nullptr, &geo);
    case 3: return tc::run<3, 128, 2, 128, 2>(planes, Gt, rows, 128, Kpad, M, b, C, s, nullptr, &geo);
    case 4: return tc::run<4, 128, 2, 128, 2>(planes, Gt, rows, 128, Kpad, M, b, C, s, nullptr, &geo);
    default: return NE_ENOTSUP;
  }
}

// The GEMM with the fused disentangle + check epilogue: M in {3, 4, 8} and
// L = 2; NE_ENOTSUP otherwise (the caller then runs the separate pass).
ne_status launch_gemm_tc_check(int M, int L, int b, const int8_t* planes, const int8_t* Bt, int64_t rows,
                               int64_t cols, int64_t K, const ne_streams& C, const ne_cstreams& dr,
                               const ne_streams& dor, uint32_t* bitmap, ne_diag* diag, int* cnt, int l,
                               cudaStream_t s) {
  const tc::ChkArgs chk{dr, dor, bitmap, diag, cnt, l};
  switch (M) {
    case 3: return gemm_tc_dispatch<3>(M, L, b, planes, Bt, rows, cols, K, C, s, &chk);
    case 4: return gemm_tc_dispatch<4>(M, L, b, planes, Bt, rows, cols, K, C, s, &chk);
    case 8: return gemm_tc_dispatch<8>(M, L, b, planes, Bt, rows, cols, K, C, s, &chk);
    default: return NE_ENOTSUP;
  }
}

}  // namespace ne
