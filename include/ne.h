/*
 * ne.h — C ABI of the B200 numerical-entanglement hot path (libne.so).
 *
 * Method: Anam & Andreopoulos, "Reliable Linear, Sesquilinear and Bijective
 * Operations on Integer Data Streams via Numerical Entanglement",
 * arXiv 1604.04740.  "P:L" cites line L of the paper text; the
 * readings of garbled passages (R1..R17) are listed in DESIGN.md.
 *
 * Pipeline (Fig. 3):  c --entangle--> eps --LSB op--> delta
 *                                  --disentangle + check / recover--> d_hat
 *
 * Conventions for every call
 * --------------------------
 * Ownership  All element pointers are DEVICE pointers allocated and owned by
 *            the caller (PyTorch in this repo).  libne never allocates, frees
 *            or synchronises; every call only enqueues kernels on `stream`
 *            and returns.  Workspaces are sized by a query call and owned by
 *            the caller.
 * Layout     SoA: a stream set is an array of M device pointers, one
 *            contiguous stream each (ne_streams / ne_cstreams /
 *            ne_cstreams32, passed BY VALUE, M <= NE_MAX_M).  "AoS" buffers
 *            interleave the M streams position-major: x[n*M + m].  Matrices
 *            are row-major and dense.  Every stream pointer must be 16-byte
 *            aligned (128-bit vector access) or the call returns NE_EINVAL.
 * Words      w = 64: entangled and output values are int64 held in
 *            64-bit two's-complement containers; plain
 *            inputs are int32.  The ne_*_w32 calls are the paper's own w = 32
 *            instantiation on int32 containers; every other call
 *            requires cfg->w == 64 (NE_ECONFIG otherwise).  LSB ops wrap mod 2^64, which is exact for
 *            every certified (in-range) result (reading R9).
 * Errors     Two channels.  (1) The returned ne_status, synchronous: argument
 *            and configuration errors, and CUDA launch errors
 *            (cudaGetLastError) as NE_ECUDA.  (2) Data-dependent outcomes —
 *            range violations of the inputs and positions flagged
 *            by the reliability check — are
 *            accumulated into a caller-owned DEVICE struct ne_diag, read by
 *            the caller after synchronising.  Reset it with ne_diag_reset.
 * Threading  No global mutable state; all calls are re-entrant.
 */
#ifndef NE_H
#define NE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NE_MAX_M 32

typedef struct cudaStream_st* ne_stream_t; /* == cudaStream_t; NULL = legacy default stream */

/* (M, w, l, k): M streams, w-bit words, shift l, guard k (Eq. 12). */
typedef struct {
  int32_t M, w, l, k;
} ne_config;

typedef enum {
  NE_OK = 0,
  NE_EINVAL = 1,          /* bad pointer, alignment, size or stream count          */
  NE_ECONFIG = 2,         /* infeasible or unsupported (M, w, l, k)               */
  NE_ERANGE = 3,          /* certification: the op's output bound exceeds range  */
  NE_EINDEX = 4,          /* excluded stream r outside [0, M)                     */
  NE_EUNRECOVERABLE = 5,  /* more than one stream absent for recovery             */
  NE_ECUDA = 6,           /* a CUDA launch failed                                 */
  NE_ENOTSUP = 7          /* shape not supported by the selected kernel           */
} ne_status;

typedef struct { int64_t* s[NE_MAX_M]; } ne_streams;
typedef struct { const int64_t* s[NE_MAX_M]; } ne_cstreams;
typedef struct { const int32_t* s[NE_MAX_M]; } ne_cstreams32;
typedef struct { int32_t* s[NE_MAX_M]; } ne_streams32;   /* w = 32 containers (ne_*_w32) */

/* Device-resident diagnostics (SPEC error list: range error naming (m,n),
 * fault positions).  first_* are INT64_MAX when nothing was recorded. */
typedef struct {
  unsigned long long range_violations; /* inputs with |c| > hi (a0)              */
  long long first_bad;                 /* min flat index m*n_total + n of those  */
  unsigned long long fault_positions;  /* positions flagged by the check (a5)    */
  long long first_fault;               /* min flagged position                   */
} ne_diag;

/* GEMM algorithms: the tcgen05 int8-digit path; CUDA-core 64 x 32-bit
 * multiply-adds for any int64 A (IMAD64); CUDA-core 32 x 32 -> 64-bit
 * IMAD.WIDE when every A entry fits int32 (IMAD32W; an entry that does not
 * is a range violation in diag). */
typedef enum { NE_GEMM_TC_I8 = 0, NE_GEMM_IMAD64 = 1, NE_GEMM_IMAD32W = 2 } ne_gemm_algo;
/* which tensor-core kernel a limb GEMM launch runs (ne_gemm_kernel_for) */
typedef enum { NE_GEMM_KERNEL_CTA = 0, NE_GEMM_KERNEL_PAIR = 1 } ne_gemm_kernel;
typedef enum { NE_OP_SCALE = 0, NE_OP_ADD = 1, NE_OP_LINEAR = 2, NE_OP_PERMUTE = 3 } ne_op_kind;

/* ======================================================== a0: host only === */

/* (l, k) maximising (M-2)l + k subject to (M-1)l + k <= w and 1 <= k <= l
 * (Eq. 12; Table II); ties -> larger l (reading R5).
 * Errors: NE_ECONFIG if M < 3, M > NE_MAX_M or infeasible; NE_EINVAL if out NULL. */
ne_status ne_config_for(int32_t M, int32_t w, ne_config* out);

/* Admissible output range [-hi, hi]: min(Eq. 13, Eq. 11
 * when M = 3) (reading R6).  Errors: NE_ECONFIG for an invalid config. */
ne_status ne_dynamic_range(const ne_config* cfg, int64_t* hi);

/* Worst-case output bound of one LSB op on inputs bounded by in_bound
 * (Remark 2): SCALE -> in*|s|, ADD -> in + max|g|, LINEAR
 * (inner/conv/gemm row) -> in * ||g||_1, PERMUTE -> in.  *out_bound gets the
 * bound; returns NE_ERANGE if it exceeds the dynamic range (chain ops by
 * feeding out_bound back in). */
ne_status ne_certify(const ne_config* cfg, ne_op_kind op, int64_t in_bound, int64_t operand,
                     int64_t* out_bound);

/* Number of balanced signed base-2^8 limbs that represent every entangled
 * value (2^l + 1) * in_bound exactly (the GEMM operand split). */
int32_t ne_gemm_limbs_for(const ne_config* cfg, int64_t in_bound);

/* The cheapest exact digit plan for the GEMM operand: returns L and sets
 * *limb_bits = b with eps = sum_{i<L} 2^(b i) d_i, every d_i in [-128, 127].
 * b = l, L = 2 when |c| <= 127 and l >= 8 (an entangled value is then exactly
 * its two int8 halves c_m, c_{m-1}); else b = 8, L = ne_gemm_limbs_for(). */
int32_t ne_gemm_limb_plan(const ne_config* cfg, int64_t in_bound, int32_t* limb_bits);

/* Fill a device ne_diag with {0, INT64_MAX, 0, INT64_MAX}. */
ne_status ne_diag_reset(ne_diag* diag, ne_stream_t stream);

/* ============================================== a1/a2: entanglement ====== */

/* Eq. 15 with the circulant operator of Eq. 14 (Eq. 7 for M = 3):
 *   eps_m[n] = c_m[n] + S_l{ c_{(m-1) mod M}[n] },  0 <= n < n_total.
 * c: M int32 streams (read once each).  eps: M int64 streams (may NOT alias c).
 * Fused range assertion (a0): every |c_m[n]| <= hi, else diag.range_violations
 * is incremented and diag.first_bad = min(m*n_total + n).  diag may be NULL. */
ne_status ne_entangle(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, ne_streams eps,
                      ne_diag* diag, ne_stream_t stream);

/* `sets` independent stream sets in one launch: set s is c.s[s*M .. s*M+M-1]
 * -> eps.s[s*M .. s*M+M-1], each entangled by Eq. 15 on its own (the C1 chain
 * entangles its operand set and its addend set together); first_bad =
 * (s*M + m)*n_total + n.  sets*M <= NE_MAX_M. */
ne_status ne_entangle_sets(const ne_config* cfg, ne_cstreams32 c, int32_t sets, int64_t n_total,
                           ne_streams eps, ne_diag* diag, ne_stream_t stream);

/* Same values, written position-major ("AoS"): eps_aos[n*M + m] — M int64 of
 * one position share DRAM sectors, so a gather by a permutation touches one
 * sector per position for M = 4.  eps_aos: 16-B aligned. */
ne_status ne_entangle_aos(const ne_config* cfg, ne_cstreams32 c, int64_t n_total,
                          int64_t* eps_aos, ne_diag* diag, ne_stream_t stream);

/* Same values, written as L balanced signed base-2^b digit planes, b =
 * limb_bits (the int8 operand of the tensor-core GEMM):
 * planes[((m*L) + i)*n_total + n] = d_i with eps = sum_i 2^(b i) d_i,
 * d_i in [-128, 127].  A value that L such digits cannot represent counts as a
 * range violation.  n_total must be a multiple of 16; 8 <= limb_bits <= 63. */
ne_status ne_entangle_limbs(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t L,
                            int32_t limb_bits, int8_t* planes, ne_diag* diag, ne_stream_t stream);

/* One stream only (the per-GPU entanglement of the one-stream-per-GPU layout,
 * P:608-611): eps_m[n] = c_m[n] + S_l{ c_prev[n] } with c_prev = c_{(m-1) mod M}.
 * Range check covers c_m only (first_bad = m*n_total + n). */
ne_status ne_entangle_stream(const ne_config* cfg, int32_t m, const int32_t* c_m,
                             const int32_t* c_prev, int64_t* eps_m, int64_t n_total,
                             ne_diag* diag, ne_stream_t stream);

/* One stream, in the int8 digit-plane format of ne_entangle_limbs:
 * planes_m[i*n_total + n] = digit i of c_m[n] + S_l{c_prev[n]}.  n_total % 16 == 0.
 * Range violations (|c_m| > hi or not representable in L digits) name m*n_total + n. */
ne_status ne_entangle_limbs_stream(const ne_config* cfg, int32_t m, const int32_t* c_m,
                                   const int32_t* c_prev, int64_t n_total, int32_t L, int32_t limb_bits,
                                   int8_t* planes_m, ne_diag* diag, ne_stream_t stream);

/* Footnote P:507-511: the shared operand of +/- self-entangled,
 * g_ent[n] = S_l{g[n]} + g[n]. */
ne_status ne_entangle_shared(const ne_config* cfg, const int32_t* g, int64_t* g_ent,
                             int64_t n_total, ne_stream_t stream);

/* ========================================= a3: LSB ops on entangled data === */
/* Eq. 9: delta_m = eps_m op g, the same routine on every stream
 * (P:380-386).  All arithmetic wraps mod 2^64.                              */

/* Element-wise x (Eq. 2 "x"): x_m[n] *= (g ? g[n] : s), in place. */
ne_status ne_op_scale(const ne_config* cfg, ne_streams x, int64_t n_total, int64_t s,
                      const int32_t* g_or_null, ne_stream_t stream);

/* Element-wise +/- (Eq. 2 "+,-"): x_m[n] += sign * a_m[n], in place, with the
 * addend already entangled (ne_entangle, or ne_entangle_shared broadcast by
 * passing the same pointer M times) (reading R10).  sign = +1/-1. */
ne_status ne_op_add(const ne_config* cfg, ne_streams x, ne_cstreams addend, int64_t n_total,
                    int32_t sign, ne_stream_t stream);

/* ne_op_scale then ne_op_add in one pass: x_m[n] = x_m[n] * (g ? g[n] : s)
 * + sign * addend_m[n] (the C1 chain's two ops; mod 2^64, in place). */
ne_status ne_op_scale_add(const ne_config* cfg, ne_streams x, int64_t n_total, int64_t s,
                          const int32_t* g_or_null, ne_cstreams addend, int32_t sign, ne_stream_t stream);

/* Op + check fused (BASELINE north star: extract and check fused into the
 * consumer kernel): ne_op_scale_add (resp. ne_op_conv) on every stream, delta
 * stored to x (resp. out) as the unfused op does, then Eqs. 16-19 + 21 run on
 * the values the kernel holds: d_out / bitmap / diag exactly as
 * ne_disentangle_check(delta, r) (bit-identical; tests compare both).  Every
 * stream's delta comes from that stream's operand only, so a fault in one
 * stream's computation still corrupts one delta (Props 2/4).  M in {3, 4, 8}
 * fused; other M run the two calls back to back.  Errors as the two calls. */
ne_status ne_op_scale_add_check(const ne_config* cfg, ne_streams x, int64_t n_total, int64_t s,
                                const int32_t* g_or_null, ne_cstreams addend, int32_t sign, int32_t r,
                                ne_streams d_out, uint32_t* bitmap, ne_diag* diag, ne_stream_t stream);
ne_status ne_op_conv_check(const ne_config* cfg, ne_cstreams x, int64_t n_total, const int32_t* g,
                           int32_t taps, int32_t correlate, ne_streams out, int32_t r, ne_streams d_out,
                           uint32_t* bitmap, ne_diag* diag, ne_stream_t stream);

/* Blocked inner product <.,.> (Eq. 2): out_m[b] = sum_{i in block b}
 * x_m[i] * v[i mod vlen], b < ceil(n_total/block) (ragged last block). */
ne_status ne_op_inner(const ne_config* cfg, ne_cstreams x, int64_t n_total, const int32_t* v,
                      int64_t vlen, int64_t block, ne_streams out, ne_stream_t stream);

/* One stream of the fused permutation + blocked inner product (the C4
 * stream-per-GPU placement; bijection P:253-258, reading R11;
 * inner product Eq. 2, reading R14): for output blocks b in
 * [b_begin, b_begin + b_count),
 *   out_m[b - b_begin] = sum_{i in block b} x_m[perm[i]] * v[i mod vlen]
 * (wrap mod 2^64; ragged last block).  x_m: one int64 entangled stream of
 * n_total (<= INT32_MAX) positions, 16-B aligned; perm: n_total int32
 * indices (a bijection, unchecked); out_m: b_count int64.  The caller
 * gathers the M streams' block sums (all_gather) and runs
 * ne_disentangle_check on them.  Errors: NE_EINVAL for a block range outside
 * [0, ceil(n_total / block)). */
ne_status ne_op_permute_inner_stream(const ne_config* cfg, const int64_t* x_m, const int32_t* perm, int64_t n_total,
                                     const int32_t* v, int64_t vlen, int64_t block, int64_t b_begin,
                                     int64_t b_count, int64_t* out_m, ne_stream_t stream);

/* Outer product (x) (Eq. 2): out_m[i*n2 + j] = x_m[i] * h[j]. */
ne_status ne_op_outer(const ne_config* cfg, ne_cstreams x, int64_t n1, const int32_t* h,
                      int64_t n2, ne_streams out, ne_stream_t stream);

/* Circular convolution (correlate = 0) / cross-correlation (correlate = 1)
 * (reading R12): out_m[n] = sum_{j<taps} g[j] x_m[(n -/+ j) mod n_total].
 * out must not alias x. */
ne_status ne_op_conv(const ne_config* cfg, ne_cstreams x, int64_t n_total, const int32_t* g,
                     int32_t taps, int32_t correlate, ne_streams out, ne_stream_t stream);

/* Tensor-core circular convolution / correlation (NEXT-2; same definition as
 * ne_op_conv): the op as a Toeplitz GEMM on tcgen05.  Output
 * block b (outputs W b .. W b + W-1, W = `block` in {128, 256}) = W_b G^T with
 * W_b[k] = x[(W b + k - s0) mod N] (s0 = taps-1 for conv, 0 for correlation)
 * and the W x Kpad int8 tap matrix G[i][k] = g[i + s0 - k] (conv) / g[k - i]
 * (corr), Kpad = roundup(taps + W - 1, 128).  x is held as L int8 digit
 * planes (base 2^limb_bits, as ne_entangle_limbs), each circularly extended to
 * plane_len bytes so that W_b is contiguous:
 *     planes[(m*L + d)*plane_len + t] = digit d of eps_m[(t - s0) mod N].
 *   ne_conv_geometry      -> the block width for (taps, L) (256 when taps >= 256
 *                            and L <= 2, else 128), Kpad and plane_len; pass the
 *                            same block to the three calls below.
 *   ne_entangle_limbs_conv : c (M int32 streams) -> entangled extended digit
 *                            planes (Eq. 15), range assertion as ne_entangle_limbs
 *                            (each position counted once, first_bad = m*N + n).
 *   ne_conv_prep_taps     : g (taps int32, each in [-128, 127], else a range
 *                            violation naming the tap) -> Gt [block][Kpad] int8.
 *   ne_op_conv_limbs      : out_m[n], n < n_total, int64 (wraps mod 2^64).
 * M <= 8, Kpad < 131072 (exact int32 digit sums), block 256 needs L <= 2,
 * else NE_ENOTSUP.  planes, Gt, out: 16-B aligned device buffers owned by the
 * caller. */
ne_status ne_conv_geometry(int64_t n_total, int32_t taps, int32_t L, int32_t* block, int64_t* kpad,
                           int64_t* plane_len);
ne_status ne_entangle_limbs_conv(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t taps,
                                 int32_t correlate, int32_t L, int32_t limb_bits, int32_t block,
                                 int8_t* planes, ne_diag* diag, ne_stream_t stream);
ne_status ne_conv_prep_taps(const int32_t* g, int32_t taps, int32_t correlate, int32_t block, int8_t* Gt,
                            ne_diag* diag, ne_stream_t stream);
ne_status ne_op_conv_limbs(const ne_config* cfg, const int8_t* planes, int32_t L, int32_t limb_bits,
                           int32_t block, const int8_t* Gt, int64_t n_total, int32_t taps, int32_t correlate,
                           ne_streams out, ne_stream_t stream);

/* Permutation (bijection I -> G, reading R11), gather:
 * out_m[i] = x_m[perm[i]].  perm must be a bijection of [0, n_total). */
ne_status ne_op_permute(const ne_config* cfg, ne_cstreams x, const int32_t* perm,
                        int64_t n_total, ne_streams out, ne_stream_t stream);

/* Integer matrix product (reading R13): C_m = A_m * B for every
 * stream m, A_m rows x K (entangled, int64), B K x cols (plain int32, shared
 * kernel g, unmodified), C_m rows x cols int64.  algo NE_GEMM_IMAD64 runs on
 * the CUDA cores; NE_GEMM_TC_I8 splits A_m into L (1..8) balanced
 * base-2^limb_bits int8 digit planes (ne_gemm_limb_plan / ne_gemm_plan_for;
 * limb_bits * (L - 1) <= 63) and B into LB (1..5) balanced base-256 digit
 * planes, and runs tcgen05.mma kind::i8 with exact int32 digit accumulators,
 * recombined in int64 (wrap mod 2^64, exact for certified results;
 * DESIGN.md §7): L = 8 and LB = 5 cover every int64 operand and every int32
 * B, so no certified operand range is refused.  ws: workspace of
 * ne_gemm_workspace() bytes (TC only).  Entries of B outside the LB-digit
 * range or of A_m outside the L-limb range count in diag.range_violations
 * (TC). */
ne_status ne_gemm_workspace(const ne_config* cfg, int64_t rows, int64_t cols, int64_t K,
                            int32_t L, int32_t LB, size_t* bytes);
ne_status ne_op_gemm(const ne_config* cfg, ne_cstreams A, const int32_t* B, int64_t rows,
                     int64_t cols, int64_t K, ne_gemm_algo algo, int32_t L, int32_t limb_bits, int32_t LB,
                     ne_streams C, void* ws, size_t ws_bytes, ne_diag* diag, ne_stream_t stream);

/* The plain (unentangled) GEMM with int32 products — the narrowest native
 * baseline of the "% overhead vs plain" comparison (no
 * entanglement involved): C_m = D_m B for m < count (<= 8), D_m one int8
 * plane per stream (ne_to_limbs with L = 1) [rows][K], Bt from
 * ne_gemm_prep_b, C_m int32 [rows][cols] (exact while K * 2^14 < 2^31).  The
 * CTA-pair kernel with double-buffered TMEM; rows and cols multiples of 256,
 * K of 128 (else NE_ENOTSUP). */
ne_status ne_op_gemm_plain_i32(int32_t count, const int8_t* planes, const int8_t* Bt, int64_t rows, int64_t cols,
                               int64_t K, ne_streams32 C, ne_stream_t stream);

/* ---- General digit plans of the tensor-core GEMM (the full certified range).
 * An entangled operand eps_m = c_m + 2^l c_{m-1} (Eq. 15) and the shared B are
 * held as int8 digit planes: eps_m = sum_{i<LA} 2^a_shift[i] D_{m,i} and
 * B = sum_{j<LB} 2^(8j) B_j, so C_m = sum_i sum_j 2^(a_shift[i] + 8j)
 * (D_{m,i} B_j), each product an exact int8 x int8 -> int32 tensor-core GEMM
 * (K < 131072), recombined in int64.
 *   kind NE_PLAN_EPS:   LA digits of eps in base 2^digit_bits (a_shift[i] =
 *                       digit_bits * i): the two-digit plan (digit_bits = l,
 *                       |c| <= 127) or balanced base 256 (ne_entangle_limbs).
 *   kind NE_PLAN_SPLIT: c_m and c_{m-1} each in D = LA / 2 balanced base-256
 *                       digits, at bit weights 0, 8, .. and l, l + 8, ..
 *                       (2 ceil-digits(|c|) planes; stream m's planes carry
 *                       only stream m's operand, so a fault in one stream's
 *                       product still corrupts that delta_m alone, Props 2/4).
 * planes: [(m*LA + i)*rows*K] int8 (K contiguous); Bt: [(j*cols + col)*K]. */
typedef enum { NE_PLAN_EPS = 0, NE_PLAN_SPLIT = 1 } ne_plan_kind;
typedef struct {
  int32_t kind;        /* ne_plan_kind */
  int32_t LA;          /* A digit planes per stream, 1..8 */
  int32_t digit_bits;  /* NE_PLAN_EPS: the digit base 2^digit_bits; NE_PLAN_SPLIT: 8 */
  int32_t LB;          /* B digit planes, 1..5 (balanced base 256) */
  int32_t a_shift[8];  /* bit weight of A plane i */
} ne_gemm_plan;

/* The cheapest exact plan for |c| <= a_bound (the plain inputs of the
 * entangled operand) and |B| <= b_bound (both <= INT32_MAX): fewest A planes,
 * the two-digit plan first, then the split plan when it needs fewer planes
 * than base-256 digits of eps.  Certification of the product (K a b <= hi) is
 * ne_certify's job.  Host-only. */
ne_status ne_gemm_plan_for(const ne_config* cfg, int64_t a_bound, int64_t b_bound, ne_gemm_plan* plan);
/* a0 + a1 into the plan's digit planes (Eq. 15; |c| <= hi and the digit
 * range asserted per value, violations named m*n_total + n).  n_total % 16 == 0. */
ne_status ne_entangle_plan(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, const ne_gemm_plan* plan,
                           int8_t* planes, ne_diag* diag, ne_stream_t stream);
/* B (K x cols int32, row-major) -> LB balanced base-256 digit planes
 * Bt[(j*cols + col)*K + k]; a value LB digits cannot hold is a range
 * violation naming k*cols + col.  K % 16 == 0, LB in [1, 5]. */
ne_status ne_gemm_prep_b_planes(const int32_t* B, int64_t K, int64_t cols, int32_t LB, int8_t* Bt, ne_diag* diag,
                                ne_stream_t stream);
/* C_m = sum_i sum_j 2^(a_shift[i] + 8j) D_{m,i} B_j for every stream: A planes
 * in groups of <= 4 TMEM accumulators, one tcgen05 launch per (group, B
 * plane), the first storing C and the others adding into it (TMA reduce-add,
 * u64 wrap).  A plain plan (LB = 1, <= 4 digits of one base) runs as
 * ne_op_gemm_limbs (CTA-pair kernel included).  Shapes as ne_op_gemm_limbs. */
ne_status ne_op_gemm_plan(const ne_config* cfg, const int8_t* planes, const ne_gemm_plan* plan, const int8_t* Bt,
                          int64_t rows, int64_t cols, int64_t K, ne_streams C, ne_stream_t stream);

/* The tensor-core GEMM on operands already in limb form: planes from
 * ne_entangle_limbs (M*L planes of rows x K int8, K contiguous) and Bt from
 * ne_gemm_prep_b (cols x K int8, K contiguous).  rows % 128 == 0,
 * cols % 128 == 0, K % 128 == 0, K < 131072 (int32 limb sums stay exact: |sum| <=
 * K * 128 * 128 must stay below 2^31, so K = 131072 itself is refused). */
ne_status ne_gemm_prep_b(const int32_t* B, int64_t K, int64_t cols, int8_t* Bt, ne_diag* diag,
                         ne_stream_t stream);
ne_status ne_op_gemm_limbs(const ne_config* cfg, const int8_t* planes, int32_t L, int32_t limb_bits,
                           const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, ne_streams C,
                           ne_stream_t stream);

/* ne_op_gemm_limbs followed by ne_disentangle_check(C, r, d_out, bitmap,
 * diag) on its outputs, fused into the GEMM epilogue: the M
 * streams' tiles of each output tile are computed back to back; the CTA that
 * stores the last of them reads the M delta tiles back (L2) and disentangles
 * and checks them (Eqs. 16-19, 21).  C (delta) is still written in full (it
 * is what recovery reads).  Results, bitmap and diag are bit-identical to the
 * unfused pair.  tile_counters: ne_gemm_check_workspace() bytes of device
 * memory, zeroed by the caller once; every call leaves them zeroed (do not
 * share one buffer between concurrently running calls).  Fused for M in
 * {3, 4, 8} and L = 2; other (M, L) run the two kernels back to back.
 * Shapes as ne_op_gemm_limbs.  Errors: NE_EINDEX if r outside [0, M). */
ne_status ne_gemm_check_workspace(int64_t rows, int64_t cols, size_t* bytes);
ne_status ne_op_gemm_limbs_check(const ne_config* cfg, const int8_t* planes, int32_t L, int32_t limb_bits,
                                 const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, ne_streams C,
                                 int32_t r, ne_streams d_out, uint32_t* bitmap, ne_diag* diag,
                                 int32_t* tile_counters, ne_stream_t stream);

/* ne_op_gemm_limbs_stream with the position-major exchange fused into the
 * epilogue (C5; one stream per GPU): the output
 * C_m (rows x cols int64, row-major) is split into ndest row blocks of
 * rows / ndest rows — exactly the contiguous position chunks j of the check's
 * all-to-all — and block j is stored by TMA straight into dests.s[j], a
 * [rows / ndest][cols] int64 region that may live in another GPU's memory
 * (a peer-mapped / symmetric-memory address reached over NVLink) or locally.
 * The stores are asynchronous bulk copies issued tile by tile while later
 * tiles are still being multiplied, so the exchange overlaps the GEMM.  If
 * C_local is non-NULL the whole C_m is also stored there (rows x cols int64,
 * local memory): the sender's copy that a recovery exchange among survivors
 * needs after a fail-stop.  The caller orders the receivers' reads after the
 * launch (stream order plus a cross-GPU barrier).  ndest in [1, 8],
 * rows % (128 ndest) == 0 (else NE_ENOTSUP); other shapes and errors as
 * ne_op_gemm_limbs_stream. */
ne_status ne_op_gemm_limbs_scatter(const ne_config* cfg, const int8_t* planes_m, int32_t L, int32_t limb_bits,
                                   const int8_t* Bt, int64_t rows, int64_t cols, int64_t K, ne_streams dests,
                                   int32_t ndest, int64_t* C_local, ne_stream_t stream);

/* Which tcgen05 kernel ne_op_gemm_limbs / ne_op_gemm (TC) launches for this
 * shape and digit plan (host-only query, no GPU needed; the same gate the
 * launch uses): *kernel = NE_GEMM_KERNEL_PAIR for the CTA-pair kernel
 * (k_gemm_pair; rows and cols multiples of 256, K of 128, M <= 8, b <= 31):
 * L = 2 limb-major passes when 4096 <= K <= 8192, or K >= 2048 with >= 256
 * pair tiles; L = 1 double-buffered tiles when K >= 1024 with >= 64 pair
 * tiles), else NE_GEMM_KERNEL_CTA (k_gemm_tc, single-CTA tiles).  The gemm trace hook
 * (ne_gemm_trace), when on, forces the single-CTA kernel.  Errors as
 * ne_op_gemm_limbs (NE_ENOTSUP for shapes the tensor-core path refuses). */
ne_status ne_gemm_kernel_for(const ne_config* cfg, int32_t L, int32_t limb_bits, int64_t rows, int64_t cols,
                             int64_t K, int32_t* kernel);

/* Debug hook (not on the hot path): every later tensor-core GEMM / Toeplitz
 * conv launch in this process records, for CTA c and its t-th tile (t < 32),
 * the %globaltimer value when the tile's accumulators are complete and when
 * its epilogue has staged the last chunk, at buf[(c * 32 + t) * 2 + {0, 1}]
 * (device memory of grid x 64 int64, zeroed by the caller).  max_clusters > 0
 * caps the persistent grid (0: occupancy-sized) — of the CTA-pair kernel too
 * (in pairs), which runs only while buf is NULL (the trace records the
 * single-CTA kernel).  buf = NULL, max_clusters = 0
 * turn it off.  Not thread-safe; NE_EINVAL if max_clusters < 0. */
ne_status ne_gemm_trace(long long* buf, int32_t max_clusters);

/* The CTA-pair kernel's schedule for two-digit GEMMs (host-only, no GPU
 * needed): of n_tiles 256 x 256 pair tiles (over all M streams) on npairs
 * resident SM pairs, *n_whole run whole; a last partial wave of r =
 * n_tiles mod npairs tiles with 2 r <= npairs runs as 2 r half tiles of
 * 256 x 128 (N = 128 MMAs, ~0.76 of a tile's time each), the same exact
 * products.  C3: 768 tiles on 74 pairs -> 740 whole + 56 halves.  One-digit
 * launches and the Toeplitz conv keep whole tiles.  NE_EINVAL for a null
 * output, n_tiles < 0 or npairs < 1. */
ne_status ne_gemm_pair_schedule(int64_t n_tiles, int64_t npairs, int64_t* n_whole);

/* Debug hook (tests): mode 0 restores the schedule above, 1 keeps every pair
 * tile whole, 2 halves every tile, for later two-digit CTA-pair launches in
 * this process.  Not thread-safe; NE_EINVAL outside 0..2. */
ne_status ne_gemm_pair_halves(int32_t mode);

/* One stream of ne_op_gemm_limbs (the per-GPU GEMM of the one-stream-per-GPU
 * layout): C_m = sum_i 2^(8i) D_{m,i} B from planes_m (L planes). */
ne_status ne_op_gemm_limbs_stream(const ne_config* cfg, const int8_t* planes_m, int32_t L,
                                  int32_t limb_bits, const int8_t* Bt, int64_t rows, int64_t cols, int64_t K,
                                  int64_t* C_m, ne_stream_t stream);

/* ====================================== a4-a6: disentangle, check, recover === */

/* Eqs. 16-19 (readings R1-R3) excluding stream r, then the
 * reliability check of Eq. 21 (Eq. 20 for M = 3), at every
 * position, in exact 2w-bit (int128) arithmetic:
 *   d_out_m[n]  = low 64 bits of the disentangled d_hat_m[n]
 *   flag[n]     = delta_r[n] != d_hat_r[n] + S_l{ d_hat_{(r-1) mod M}[n] }
 * bitmap (nullable): bit (n mod 32) of word n/32 = flag[n] (ceil(n_total/32)
 * words, fully written).  diag (nullable): fault_positions += #flags,
 * first_fault = min flagged n.  Errors: NE_EINDEX if r outside [0, M). */
ne_status ne_disentangle_check(const ne_config* cfg, ne_cstreams delta, int64_t n_total,
                               int32_t r, ne_streams d_out, uint32_t* bitmap, ne_diag* diag,
                               ne_stream_t stream);

/* Fail-stop recovery (Props 1/3): Eqs. 16-19 excluding
 * the absent stream r (delta.s[r] == NULL, never read).  Errors:
 * NE_EUNRECOVERABLE if any other delta.s[m] is NULL. */
ne_status ne_recover(const ne_config* cfg, ne_cstreams delta, int64_t n_total, int32_t r,
                     ne_streams d_out, ne_stream_t stream);

/* Fused permutation + blocked inner product + disentangle/check (the C4 hot
 * path): for block b, delta_m[b] = sum_{i<block} x_m[perm[b*block+i]] * v[i mod vlen]
 * (perm NULL = identity), then d_out / bitmap / diag exactly as
 * ne_disentangle_check on delta (r excluded).  x is AoS (x_aos[n*M + m],
 * aos = 1) or SoA (x.s[m], aos = 0).  delta_out (nullable) receives delta. */
ne_status ne_op_permute_inner_check(const ne_config* cfg, ne_cstreams x, const int64_t* x_aos,
                                    int32_t aos, const int32_t* perm, int64_t n_total,
                                    const int32_t* v, int64_t vlen, int64_t block, int32_t r,
                                    ne_streams delta_out, ne_streams d_out, uint32_t* bitmap,
                                    ne_diag* diag, ne_stream_t stream);

/* The same op as a partitioned scatter-reduce, without a random DRAM gather
 * (k_permute_bucket.cu): the pairs (i, perm[i]) are partitioned into cells
 * (source window perm[i] >> S, destination range of output blocks) by one
 * scatter pass over perm (coalesced; a chunk's pairs sorted in shared
 * memory); then one CTA per destination range walks its cells window by
 * window — every CTA reads the same window of x, which stays in L2 — and
 * adds each pair's M products x_m[perm[i]] * v[i mod vlen] into its block
 * sums (int64 sums mod 2^64, so delta is bit-identical to the gather form),
 * written once; then ne_disentangle_check on delta.  Two plans (which one:
 * ne_permute_inner_plan): owned runs (each block's pairs one run per cell,
 * each block summed by one thread, no atomics; power-of-two blocks dividing
 * 4096) or shared-memory block sums with 32-bit shared atomics.  x AoS only (x_aos[n*M + m], 16-byte
 * aligned), M <= 8 (NE_ENOTSUP otherwise), perm required and a bijection of
 * [0, n_total): entries outside it are range violations in diag (first_bad =
 * i) and skipped.  delta (required) receives the block sums.  workspace:
 * device memory of at least ne_permute_inner_workspace(cfg, n_total, block)
 * bytes, 16-byte aligned, owned by the caller (NE_EINVAL if smaller). */
ne_status ne_permute_inner_workspace(const ne_config* cfg, int64_t n_total, int64_t block, size_t* bytes);

/* The plan ne_op_permute_inner_check_bucketed runs for (cfg->M, n_total,
 * block); host only, no device work.  mode 1 = owned runs (the C4 default:
 * block a power of two dividing the 4096-position scatter chunk, at least 2
 * positions per run-index entry): a chunk's slice of a cell is sorted by
 * (window, output block), a pair is packed in 32 bits ((i mod block) << S |
 * perm[i] mod 2^S), one 32-bit run-index entry per (cell, block) holds the
 * run's offset and length, and reduce thread t owns blocks t, t + T, ... of
 * its range and sums their runs in registers — no atomics; mode 0 = 8-byte
 * pairs and shared-memory block sums (two 32-bit shared atomics per
 * product).  Outputs (each nullable): S (2^S entries of x per window), nwin
 * windows, nrange destination ranges (= reduce CTAs), rb output blocks per
 * range, cap pair slots per cell, index_bytes (run index; 0 in mode 0).
 * NE_EINVAL for n_total < 0 or > INT32_MAX or block < 1. */
ne_status ne_permute_inner_plan(const ne_config* cfg, int64_t n_total, int64_t block, int32_t* mode, int32_t* S,
                                int32_t* nwin, int32_t* nrange, int64_t* rb, int64_t* cap, int64_t* index_bytes);
ne_status ne_op_permute_inner_check_bucketed(const ne_config* cfg, const int64_t* x_aos, const int32_t* perm,
                                             int64_t n_total, const int32_t* v, int64_t vlen, int64_t block,
                                             int32_t r, ne_streams delta, ne_streams d_out, uint32_t* bitmap,
                                             ne_diag* diag, void* workspace, size_t ws_bytes,
                                             ne_stream_t stream);

/* ====================================== comparison baseline: ABFT (NEXT-1) === */
/* The paper's comparison method, run on the same hardware so the
 * overhead of entanglement can be compared with ABFT's at equal fault
 * tolerance (one faulty stream of M+1 detected, one lost stream recovered).  */

/* Eq. 4: r_out[n] = sum_m c_m[n] (int32; a sum that does not fit
 * — ABFT's extra ceil(log2 M) bits, Table I — is a range violation naming n). */
ne_status ne_abft_encode(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t* r_out,
                         ne_diag* diag, ne_stream_t stream);
/* Plain int32 streams x[0..count) -> L balanced int8 digit planes
 * planes[(s*L + i)*n_total + n] (the tensor-core operand of unentangled data;
 * a value L digits cannot hold is a range violation).  n_total % 16 == 0. */
ne_status ne_to_limbs(ne_cstreams32 x, int32_t count, int64_t n_total, int32_t L, int8_t* planes,
                      ne_diag* diag, ne_stream_t stream);
/* Eqs. 4-5 in tensor-core form, one pass: pdata[m*n_total + n] = c_m[n] as one
 * int8 digit, psum[j*n_total + n] = base-256 digit j (Ls digits) of
 * r = sum_m c_m.  Values that do not fit are range violations (data: m*n + n,
 * checksum: M*n + n).  n_total % 16 == 0, 1 <= Ls <= 4. */
ne_status ne_abft_encode_limbs(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int8_t* pdata,
                               int32_t Ls, int8_t* psum, ne_diag* diag, ne_stream_t stream);
/* ABFT on the tensor-core convolution (the paper's conv comparison, P:1102-
 * 1116): plain data as one int8 digit plane per stream and the checksum r =
 * sum_m c_m (Eq. 4) as Ls base-256 digit planes, circularly extended exactly
 * like ne_entangle_limbs_conv (same block / plane_len); out-of-range values
 * are range violations (data m*N + n, checksum M*N + n).  Then
 * ne_op_conv_limbs_plain runs the Toeplitz conv on `count` plane sets of L
 * digits (count <= 8; no entanglement config involved), and ne_abft_check /
 * ne_abft_recover finish.  Layout, alignment and limits as the conv calls. */
ne_status ne_abft_encode_conv(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t taps,
                              int32_t correlate, int32_t block, int8_t* pdata, int32_t Ls, int8_t* psum,
                              ne_diag* diag, ne_stream_t stream);
ne_status ne_op_conv_limbs_plain(int32_t count, const int8_t* planes, int32_t L, int32_t limb_bits,
                                 int32_t block, const int8_t* Gt, int64_t n_total, int32_t taps,
                                 int32_t correlate, ne_streams out, ne_stream_t stream);
/* Eq. 6: flag[n] = (sum_m d_m[n] != e[n]) mod 2^64, bitmap/diag as
 * ne_disentangle_check. */
ne_status ne_abft_check(const ne_config* cfg, ne_cstreams d, const int64_t* e, int64_t n_total,
                        uint32_t* bitmap, ne_diag* diag, ne_stream_t stream);
/* d_r = e - sum_{m != r} d_m (d.s[r] may be NULL; any other NULL ->
 * NE_EUNRECOVERABLE). */
ne_status ne_abft_recover(const ne_config* cfg, ne_cstreams d, const int64_t* e, int64_t n_total,
                          int32_t r, int64_t* d_r, ne_stream_t stream);

/* ============================== w = 32 containers (NEXT-3; Table II) === */
/* The same operations with cfg->w == 32 (e.g. ne_config_for(3, 32) = (l, k) =
 * (11, 10), dynamic range +-1 046 528): entangled values and results in int32
 * containers, every op mod 2^32, the 2w-bit temporaries of Eqs. 16-19/21 in
 * int64 (exact: |t| < 2^63, (M-1) l <= 31).  d_out gets the low 32 bits of the
 * exact d_hat (reading R17).  Layout, bitmap, diag and errors as the w = 64
 * calls; NE_ECONFIG unless cfg->w == 32.                                      */
ne_status ne_entangle_w32(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, ne_streams32 eps,
                          ne_diag* diag, ne_stream_t stream);
ne_status ne_entangle_sets_w32(const ne_config* cfg, ne_cstreams32 c, int32_t sets, int64_t n_total,
                               ne_streams32 eps, ne_diag* diag, ne_stream_t stream);
/* x_m[n] = x_m[n] * (g ? g[n] : s) + sign * addend_m[n] (addend_or_null: a host
 * pointer to the entangled addend set, or NULL for scale only), in place. */
ne_status ne_op_scale_add_w32(const ne_config* cfg, ne_streams32 x, int64_t n_total, int32_t s,
                              const int32_t* g_or_null, const ne_cstreams32* addend_or_null, int32_t sign,
                              ne_stream_t stream);
ne_status ne_op_scale_add_check_w32(const ne_config* cfg, ne_streams32 x, int64_t n_total, int32_t s,
                                    const int32_t* g_or_null, ne_cstreams32 addend, int32_t sign, int32_t r,
                                    ne_streams32 d_out, uint32_t* bitmap, ne_diag* diag, ne_stream_t stream);
ne_status ne_disentangle_check_w32(const ne_config* cfg, ne_cstreams32 delta, int64_t n_total, int32_t r,
                                   ne_streams32 d_out, uint32_t* bitmap, ne_diag* diag, ne_stream_t stream);
ne_status ne_recover_w32(const ne_config* cfg, ne_cstreams32 delta, int64_t n_total, int32_t r,
                         ne_streams32 d_out, ne_stream_t stream);
/* as ne_inject_sweep with 32 bits per word: trial t = (s*window + n)*32 + bit;
 * flagwords / dhat: M*window*32 entries (dhat times M, int32). */
ne_status ne_inject_sweep_w32(const ne_config* cfg, ne_cstreams32 delta, int64_t window, int32_t r,
                              uint64_t* flagwords, int32_t* dhat, ne_stream_t stream);
/* The C4 class at w = 32 (permute + inner, where the range
 * allows: every block sum must lie inside ne_dynamic_range).  AoS containers
 * x_aos[n*M + m] = eps_m[n] (int32; M = 4: 16 bytes per position, one 128-bit
 * load in the random gather).  ne_entangle_aos_w32: Eq. 15 mod 2^32, inputs
 * outside the dynamic range counted as in ne_entangle_w32 (first_bad =
 * m*N + n).  ne_op_permute_inner_check_w32: for block b,
 * delta_m[b] = sum_{i<block} x_m[perm[b*block+i]] * v[i mod vlen] mod 2^32
 * (perm NULL = identity), then d_out / bitmap / diag exactly as
 * ne_disentangle_check_w32 on delta (r excluded); delta_out (nullable)
 * receives delta.  n_total <= INT32_MAX; NE_EINDEX if r outside [0, M). */
ne_status ne_entangle_aos_w32(const ne_config* cfg, ne_cstreams32 c, int64_t n_total, int32_t* x_aos,
                              ne_diag* diag, ne_stream_t stream);
ne_status ne_op_permute_inner_check_w32(const ne_config* cfg, const int32_t* x_aos, const int32_t* perm,
                                        int64_t n_total, const int32_t* v, int64_t vlen, int64_t block,
                                        int32_t r, ne_streams32 delta_out, ne_streams32 d_out,
                                        uint32_t* bitmap, ne_diag* diag, ne_stream_t stream);

/* ============================================== a7: fault injection (test) === */

/* x[idx] ^= mask (one 64-bit word). */
ne_status ne_inject(int64_t* x, int64_t idx, uint64_t mask, ne_stream_t stream);

/* Exhaustive single-bit sweep over the first `window` (<= 64) positions of
 * delta: trial t = (s*window + n)*64 + bit flips bit `bit` of delta_s[n] and
 * re-runs disentangle + check (r excluded) on positions 0..window-1.
 * flagwords[t] = bit p set iff position p is flagged; dhat[t*M + m] = d_out_m[n].
 * Both out arrays: M*window*64 entries (dhat: times M). */
ne_status ne_inject_sweep(const ne_config* cfg, ne_cstreams delta, int64_t window, int32_t r,
                          uint64_t* flagwords, int64_t* dhat, ne_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* NE_H */
