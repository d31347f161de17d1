/*
 * ne_oracle.c — plain CPU oracle of arXiv 1604.04740 (numerical entanglement).
 *
 * TEST INFRASTRUCTURE ONLY (see ne_oracle.h): loaded by tests/, smoke() and
 * bench.py's CPU legs; never by the product path.
 *
 * Straight transcription of the paper, in its order and notation:
 *   §III-A  Eq. 7 (entangle, M = 3), Eq. 8, Eq. 10 (disentangle), Eq. 11
 *   §III-C  Eq. 12 (constraint), Eq. 13 (range), Eqs. 14-15 (circulant E),
 *           Eqs. 16-19 (disentangle excluding r)
 *   Appendix Eq. 20 / Eq. 21 (reliability check), Props 1-4.
 * Readings of garbled passages: R1 Eq. 16 is multiplied
 * by (-1)^M; R2 Eq. 18's subscript M-1 is (r+M-1) mod M; R3 Eq. 19 runs
 * 1 <= m <= M-2; R4 Eq. 21's r ranges over 0 <= r < M; R5 ties in (l,k) go to
 * the larger l.
 */
#include "ne_oracle.h"

#include <pthread.h>
#include <stddef.h>
#include <unistd.h>

#include "../gen/ne_gen.h"

typedef __int128 i128;
typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- a0 ---- */

/* choose (l,k) maximising (M-2)l + k subject to (M-1)l + k <= w
 * (Eq. 12) and k <= l; l, k >= 1.  Ties -> larger l (reading R5). */
int32_t or_config_for(int32_t M, int32_t w, or_config* out) {
  if (M < 3 || w < 4 || w > 64) return -1;
  int32_t best_l = 0, best_k = 0, best_v = -1;
  for (int32_t l = 1; l <= w; ++l) {
    for (int32_t k = 1; k <= l; ++k) {
      if ((M - 1) * l + k > w) continue;
      int32_t v = (M - 2) * l + k;
      if (v > best_v || (v == best_v && l > best_l)) {
        best_v = v;
        best_l = l;
        best_k = k;
      }
    }
  }
  if (best_v < 0) return -1;
  out->M = M;
  out->w = w;
  out->l = best_l;
  out->k = best_k;
  return 0;
}

static i128 pow2(int32_t e) { return ((i128)1) << e; }

/* Eq. 11, M = 3: |d| <= 2^(l+k-1) - 2^l. */
int64_t or_range_eq11(const or_config* cfg) {
  i128 v = pow2(cfg->l + cfg->k - 1) - pow2(cfg->l);
  return (int64_t)v;
}

/* Eq. 13: |d| <= 2^((M-3)l+k) (2^(l-1) - 1). */
int64_t or_range_eq13(const or_config* cfg) {
  i128 v = pow2((cfg->M - 3) * cfg->l + cfg->k) * (pow2(cfg->l - 1) - 1);
  return (int64_t)v;
}

/* Conservative admissible range (reading R6): the smaller of Eq. 13 and,
 * for M = 3, Eq. 11. */
int64_t or_dynamic_range(const or_config* cfg) {
  int64_t hi = or_range_eq13(cfg);
  if (cfg->M == 3) {
    int64_t h11 = or_range_eq11(cfg);
    if (h11 < hi) hi = h11;
  }
  return hi;
}

/* w-bit two's-complement container: keep the low w bits, sign-extend. */
int64_t or_wrap(const or_config* cfg, int64_t x) {
  if (cfg->w >= 64) return x;
  uint64_t mask = (1ull << cfg->w) - 1ull;
  uint64_t u = (uint64_t)x & mask;
  if (u >> (cfg->w - 1)) u |= ~mask;
  return (int64_t)u;
}

/* w-bit sum / product: computed mod 2^64 then reduced mod 2^w. */
static int64_t wadd(const or_config* cfg, int64_t a, int64_t b) {
  return or_wrap(cfg, (int64_t)((uint64_t)a + (uint64_t)b));
}
static int64_t wmul(const or_config* cfg, int64_t a, int64_t b) {
  return or_wrap(cfg, (int64_t)((uint64_t)a * (uint64_t)b));
}
/* S_l{a} for l >= 0, as a w-bit left shift (truncating at the MSB). */
static int64_t wshl(const or_config* cfg, int64_t a, int32_t l) {
  return or_wrap(cfg, (int64_t)((uint64_t)a << l));
}

int64_t or_range_check(const int64_t* x, int64_t count, int64_t hi, int64_t* first_bad) {
  int64_t bad = 0;
  if (first_bad) *first_bad = -1;
  for (int64_t i = 0; i < count; ++i) {
    if (x[i] > hi || x[i] < -hi) {
      if (bad == 0 && first_bad) *first_bad = i;
      ++bad;
    }
  }
  return bad;
}

/* ---------------------------------------------------------------- a1/a2 - */

/* Eq. 15 with the circulant operator of Eq. 14: row m of E has
 * 1 on the diagonal and S_l at column (m-1) mod M, i.e.
 *   eps_{m,n} = c_{m,n} + S_l{c_{(m-1) mod M, n}}.
 * For M = 3 this is Eq. 7. */
void or_entangle(const or_config* cfg, const int64_t* c, int64_t N, int64_t* eps) {
  const int32_t M = cfg->M;
  for (int32_t m = 0; m < M; ++m) {
    const int32_t prev = (m + M - 1) % M;
    for (int64_t n = 0; n < N; ++n) {
      eps[(int64_t)m * N + n] =
          wadd(cfg, c[(int64_t)m * N + n], wshl(cfg, c[(int64_t)prev * N + n], cfg->l));
    }
  }
}

/* Footnote P:507-511: for op in {+,-}, g_n <- S_l{g_n} + g_n. */
void or_entangle_shared(const or_config* cfg, const int64_t* g, int64_t N, int64_t* g_ent) {
  for (int64_t n = 0; n < N; ++n) g_ent[n] = wadd(cfg, wshl(cfg, g[n], cfg->l), g[n]);
}

/* ---------------------------------------------------------------- a3 ---- */
/* Eq. 2 / Eq. 9: delta_m = eps_m op g, unchanged
 * routine on every stream.  Definitions (DESIGN.md §"Op definitions"). */

/* element-by-element x (scalar s, or g_n if g is given) */
void or_op_scale(const or_config* cfg, int64_t* x, int64_t rows, int64_t N, int64_t s,
                 const int64_t* g_or_null) {
  for (int64_t m = 0; m < rows; ++m)
    for (int64_t n = 0; n < N; ++n) {
      int64_t f = g_or_null ? g_or_null[n] : s;
      x[m * N + n] = wmul(cfg, x[m * N + n], f);
    }
}

/* element-by-element +/- with a same-shaped addend a (already entangled when
 * x is entangled: reading R10) */
void or_op_add(const or_config* cfg, int64_t* x, const int64_t* a, int64_t rows, int64_t N,
               int32_t sign) {
  for (int64_t m = 0; m < rows; ++m)
    for (int64_t n = 0; n < N; ++n) {
      int64_t v = a[m * N + n];
      x[m * N + n] = sign >= 0 ? wadd(cfg, x[m * N + n], v)
                               : or_wrap(cfg, (int64_t)((uint64_t)x[m * N + n] - (uint64_t)v));
    }
}

/* blocked inner product <.,.>: out_{m,b} = sum_{i in block b} x_{m,i} v_{i mod vlen}
 * (reading R14: vlen = block gives one shared vector per block). */
void or_op_inner(const or_config* cfg, const int64_t* x, int64_t rows, int64_t N,
                 const int64_t* v, int64_t vlen, int64_t block, int64_t* out) {
  const int64_t nb = (N + block - 1) / block;
  for (int64_t m = 0; m < rows; ++m)
    for (int64_t b = 0; b < nb; ++b) {
      int64_t acc = 0;
      for (int64_t i = b * block; i < N && i < (b + 1) * block; ++i)
        acc = wadd(cfg, acc, wmul(cfg, x[m * N + i], v[i % vlen]));
      out[m * nb + b] = acc;
    }
}

/* outer product (x): out_m[i][j] = x_{m,i} h_j */
void or_op_outer(const or_config* cfg, const int64_t* x, int64_t rows, int64_t N1,
                 const int64_t* h, int64_t N2, int64_t* out) {
  for (int64_t m = 0; m < rows; ++m)
    for (int64_t i = 0; i < N1; ++i)
      for (int64_t j = 0; j < N2; ++j)
        out[(m * N1 + i) * N2 + j] = wmul(cfg, x[m * N1 + i], h[j]);
}

/* circular convolution (*) / cross-correlation with a T-tap g (P:257-259,
 * reading R12): out_{m,n} = sum_{j<T} g_j x_{m,(n -/+ j) mod N}. */
void or_op_conv(const or_config* cfg, const int64_t* x, int64_t rows, int64_t N,
                const int64_t* g, int64_t T, int32_t correlate, int64_t* out) {
  for (int64_t m = 0; m < rows; ++m)
    for (int64_t n = 0; n < N; ++n) {
      int64_t acc = 0;
      for (int64_t j = 0; j < T; ++j) {
        int64_t idx = correlate ? (n + j) % N : ((n - j) % N + N) % N;
        acc = wadd(cfg, acc, wmul(cfg, g[j], x[m * N + idx]));
      }
      out[m * N + n] = acc;
    }
}

/* integer matrix product (reading R13): C = A B with A the
 * rows_total x K stack of the stream sub-blocks, B K x cols. Naive triple loop. */
static void gemm_rows(const or_config* cfg, const int64_t* A, int64_t i0, int64_t i1, int64_t K,
                      const int64_t* B, int64_t cols, int64_t* C) {
  for (int64_t i = i0; i < i1; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      int64_t acc = 0;
      for (int64_t k = 0; k < K; ++k) acc = wadd(cfg, acc, wmul(cfg, A[i * K + k], B[k * cols + j]));
      C[i * cols + j] = acc;
    }
}

/* The outer loop may be split over threads (SURVEY §8(c) allows parallelising
 * the big GEMMs' outer loops): rows are independent and every C[i][j] is the
 * same single accumulation in the same order, so the result does not depend
 * on the thread count (or_set_threads; 1 = the single-core baseline). */
static int32_t g_threads = 1;
void or_set_threads(int32_t n) { g_threads = n > 0 ? n : 1; }
int32_t or_max_threads(void) { return (int32_t)sysconf(_SC_NPROCESSORS_ONLN); }

typedef struct {
  const or_config* cfg;
  const int64_t *A, *B;
  int64_t i0, i1, K, cols;
  int64_t* C;
} gemm_job;

static void* gemm_job_run(void* p) {
  const gemm_job* j = (const gemm_job*)p;
  gemm_rows(j->cfg, j->A, j->i0, j->i1, j->K, j->B, j->cols, j->C);
  return NULL;
}

void or_op_gemm(const or_config* cfg, const int64_t* A, int64_t rows_total, int64_t K,
                const int64_t* B, int64_t cols, int64_t* C) {
  int64_t T = g_threads < rows_total ? g_threads : rows_total;
  if (T <= 1) {
    gemm_rows(cfg, A, 0, rows_total, K, B, cols, C);
    return;
  }
  if (T > 256) T = 256;
  pthread_t th[256];
  gemm_job jobs[256];
  for (int64_t t = 0; t < T; ++t) {
    jobs[t] = (gemm_job){cfg, A, B, t * rows_total / T, (t + 1) * rows_total / T, K, cols, C};
    pthread_create(&th[t], NULL, gemm_job_run, &jobs[t]);
  }
  for (int64_t t = 0; t < T; ++t) pthread_join(th[t], NULL);
}

/* permutation (bijection I -> G, reading R11): out_m[i] = x_m[perm[i]] */
void or_op_permute(const int64_t* x, int64_t rows, int64_t N, const int64_t* perm,
                   int64_t* out) {
  for (int64_t m = 0; m < rows; ++m)
    for (int64_t i = 0; i < N; ++i) out[m * N + i] = x[m * N + perm[i]];
}

/* ---------------------------------------------------------------- a4-a6 - */

/* The disentanglement of §III-C at one position n, excluding stream r:
 *
 * Eq. 16 builds the 2w-bit d_temp from the M-1 streams other
 * than r; reading R1 multiplies it by s = (-1)^M so that M = 3 reproduces
 * Eq. 10's d_temp = delta_2 - S_l{delta_1}:
 *     t = s * sum_{m=0}^{M-2} (-1)^m S_{(M-2-m)l}{ delta_{(r+1+m) mod M} }
 * Eq. 17: d_p = S_{-[2w-(M-1)l]}{ S_{2w-(M-1)l}{t} }, p = (r+M-1) mod M,
 *     i.e. the low (M-1)l bits of t, sign-extended.
 * Eq. 18 (reading R2): d_r = S_{-(M-1)l}{ s (t - d_p) }.
 * Eq. 19 (reading R3): for m = 1..M-2,
 *     d_{(r+m) mod M} = delta_{(r+m) mod M} - S_l{ d_{(r+m-1) mod M} }.
 * Eq. 21 (reading R4; Eq. 20 for M = 3):
 *     flag = delta_r - [ d_r + S_l{ d_p } ] != 0, evaluated exactly in 2w bits.
 * All temporaries are exact int128 (the 2w-bit register of P:561-565,
 * footnote P:717-720).  Outputs are the low w bits of the exact values. */
int32_t or_disentangle_one(const or_config* cfg, const int64_t* delta, int32_t r,
                           int64_t* dhat, int32_t check) {
  const int32_t M = cfg->M, l = cfg->l;
  const int32_t b = (M - 1) * l;
  const i128 s = (M % 2 == 0) ? 1 : -1;

  /* Eq. 16 x (-1)^M */
  i128 t = 0;
  for (int32_t m = 0; m <= M - 2; ++m) {
    i128 term = (i128)delta[(r + 1 + m) % M] * pow2((M - 2 - m) * l);
    t += (m % 2 == 0) ? term : -term;
  }
  t = s * t;

  /* Eq. 17: sign-extend the low b bits of t */
  const int32_t p = (r + M - 1) % M;
  u128 low = (u128)t & (((u128)1 << b) - 1);
  i128 d_p = (i128)low;
  if (low >> (b - 1)) d_p -= pow2(b);

  /* Eq. 18: exact arithmetic right shift (floor division by 2^b) */
  i128 num = s * (t - d_p);
  i128 d_r = num >> b; /* gcc: arithmetic shift on signed __int128 */

  i128 d[64];
  d[r] = d_r;
  d[p] = d_p;
  /* Eq. 19, m = 1 .. M-2 */
  for (int32_t m = 1; m <= M - 2; ++m) {
    int32_t cur = (r + m) % M, prv = (r + m - 1) % M;
    d[cur] = (i128)delta[cur] - d[prv] * pow2(l);
  }

  for (int32_t m = 0; m < M; ++m) dhat[m] = or_wrap(cfg, (int64_t)(uint64_t)(u128)d[m]);

  if (!check) return 0;
  /* Eq. 21 (Eq. 20 for M = 3) */
  i128 resynth = d_r + d_p * pow2(l);
  return ((i128)delta[r] - resynth) != 0 ? 1 : 0;
}

int64_t or_disentangle_check(const or_config* cfg, const int64_t* delta, int64_t N,
                             int32_t r, int64_t* dhat, uint8_t* flags) {
  const int32_t M = cfg->M;
  int64_t col[64], out[64], nflag = 0;
  for (int64_t n = 0; n < N; ++n) {
    for (int32_t m = 0; m < M; ++m) col[m] = delta[(int64_t)m * N + n];
    int32_t f = or_disentangle_one(cfg, col, r, out, 1);
    for (int32_t m = 0; m < M; ++m) dhat[(int64_t)m * N + n] = out[m];
    if (flags) flags[n] = (uint8_t)f;
    nflag += f;
  }
  return nflag;
}

/* Props 1/3 (proofs P:1172-1188): the
 * same Eqs. 16-19, never reading stream r.  Error (-1) if more than one
 * stream is absent or r is not the absent one. */
int32_t or_recover(const or_config* cfg, const int64_t* const* delta, int64_t N, int32_t r,
                   int64_t* dhat) {
  const int32_t M = cfg->M;
  int32_t absent = 0;
  for (int32_t m = 0; m < M; ++m)
    if (delta[m] == NULL) {
      if (m != r) return -1;
      ++absent;
    }
  if (absent > 1) return -1;
  int64_t col[64], out[64];
  for (int64_t n = 0; n < N; ++n) {
    for (int32_t m = 0; m < M; ++m) col[m] = (m == r) ? 0 : delta[m][n];
    or_disentangle_one(cfg, col, r, out, 0);
    for (int32_t m = 0; m < M; ++m) dhat[(int64_t)m * N + n] = out[m];
  }
  return 0;
}

/* ---------------------------------------------------------------- ABFT --- */
/* The comparison method of §II-A: one extra checksum stream. */

/* Eq. 4: r_n = sum_{m=0}^{M-1} c_{m,n} */
void or_abft_encode(const or_config* cfg, const int64_t* c, int64_t N, int64_t* r_out) {
  for (int64_t n = 0; n < N; ++n) {
    int64_t acc = 0;
    for (int32_t m = 0; m < cfg->M; ++m) acc = wadd(cfg, acc, c[(int64_t)m * N + n]);
    r_out[n] = acc;
  }
}

/* Eq. 6: a fault in any single stream of the M+1 is flagged where
 * sum_{m=0}^{M-1} d_{m,n} != e_n */
int64_t or_abft_check(const or_config* cfg, const int64_t* d, const int64_t* e, int64_t N, uint8_t* flags) {
  int64_t nflag = 0;
  for (int64_t n = 0; n < N; ++n) {
    int64_t acc = 0;
    for (int32_t m = 0; m < cfg->M; ++m) acc = wadd(cfg, acc, d[(int64_t)m * N + n]);
    int32_t f = acc != e[n];
    if (flags) flags[n] = (uint8_t)f;
    nflag += f;
  }
  return nflag;
}

/* the lost stream r = e - (sum of the remaining output streams) */
int32_t or_abft_recover(const or_config* cfg, const int64_t* const* d, const int64_t* e, int64_t N, int32_t r,
                        int64_t* d_r) {
  for (int32_t m = 0; m < cfg->M; ++m)
    if ((d[m] == NULL) != (m == r)) return -1;
  for (int64_t n = 0; n < N; ++n) {
    int64_t acc = e[n];
    for (int32_t m = 0; m < cfg->M; ++m)
      if (m != r) acc = or_wrap(cfg, (int64_t)((uint64_t)acc - (uint64_t)d[m][n]));
    d_r[n] = acc;
  }
  return 0;
}

/* S:187-195 worst-case bounds */
int64_t or_certify(int32_t op, int64_t in_bound, int64_t operand) {
  switch (op) {
    case 0: return in_bound * operand;
    case 1: return in_bound + operand;
    case 2: return in_bound * operand;
    default: return in_bound;
  }
}

/* ---------------------------------------------------------------- inputs */

void or_gen_uniform(uint64_t seed, uint32_t tag, uint32_t stream, int64_t lo, int64_t hi,
                    int64_t offset, int64_t count, int64_t* out) {
  uint64_t key = ne_gen_key(seed, tag, stream);
  for (int64_t i = 0; i < count; ++i) out[i] = ne_gen_uniform(key, (uint64_t)(offset + i), lo, hi);
}

void or_gen_perm(uint64_t seed, uint32_t tag, int64_t n, int64_t offset, int64_t count,
                 int64_t* out) {
  uint64_t key = ne_gen_key(seed, tag, 0);
  for (int64_t i = 0; i < count; ++i) out[i] = (int64_t)ne_gen_perm(key, (uint64_t)n, (uint64_t)(offset + i));
}

