/*
 * ne_oracle.h — the CPU oracle for the numerical-entanglement hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load, call or execute
 * anything under oracle/.  The product path (paper_1604_04740_b200/, libne.so)
 * never links or imports it, and this code shares nothing with it except the
 * seeded input generator gen/ne_gen.h (which holds none of the method).
 *
 * Plain, slow, single-threaded C11 with __int128 for the 2w-bit temporaries.
 * Every function cites the PAPER.md passage it follows ("P:L" = line L of
 * /root/reference/PAPER.md; "S:L" = line L of SPEC.md).  Where the paper is
 * garbled the reading taken is the one listed in DESIGN.md §"Readings".
 *
 * Value convention: every integer lives in an int64_t.  A configuration with
 * word width w < 64 (w = 16 or 32, test instantiations) stores w-bit values
 * sign-extended; all arithmetic on entangled data is reduced mod 2^w
 * (or_wrap) exactly as a w-bit two's-complement machine would.
 *
 * Parity status: every function below is pinned by a `-m "not gpu"` test in
 * tests/test_oracle_*.py (see DESIGN.md §"Oracle pins"); none is unpinned.
 */
#ifndef NE_ORACLE_H
#define NE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { int32_t M, w, l, k; } or_config;

/* a0: (l,k) selection, P:637-649 (Eq. 12) and P:502-504; ties -> larger l. */
int32_t or_config_for(int32_t M, int32_t w, or_config* out);
/* a0: admissible output range [-hi, hi]: min(Eq. 13, Eq. 11 if M = 3). */
int64_t or_dynamic_range(const or_config* cfg);
/* Eq. 11 and Eq. 13 separately. */
int64_t or_range_eq11(const or_config* cfg);
int64_t or_range_eq13(const or_config* cfg);
/* reduce mod 2^w and sign-extend (the w-bit container). */
int64_t or_wrap(const or_config* cfg, int64_t x);

/* a0 range assertion: number of |x| > hi, first offending flat index (or -1). */
int64_t or_range_check(const int64_t* x, int64_t count, int64_t hi, int64_t* first_bad);

/* a1: Eq. 7 / Eq. 15, eps_m = c_m + S_l{c_(m-1) mod M}.  c, eps: M x N row-major. */
void or_entangle(const or_config* cfg, const int64_t* c, int64_t N, int64_t* eps);
/* a2: footnote P:507-511, g <- S_l{g} + g. */
void or_entangle_shared(const or_config* cfg, const int64_t* g, int64_t N, int64_t* g_ent);

/* a3: LSB ops of Eq. 2, applied row by row to `rows` streams of
 * length N, in w-bit arithmetic (w = 64 gives the plain definition in Z for
 * any certified input). */
void or_op_scale(const or_config* cfg, int64_t* x, int64_t rows, int64_t N, int64_t s,
                 const int64_t* g_or_null);
void or_op_add(const or_config* cfg, int64_t* x, const int64_t* a, int64_t rows, int64_t N,
               int32_t sign);
void or_op_inner(const or_config* cfg, const int64_t* x, int64_t rows, int64_t N,
                 const int64_t* v, int64_t vlen, int64_t block, int64_t* out);
void or_op_outer(const or_config* cfg, const int64_t* x, int64_t rows, int64_t N1,
                 const int64_t* h, int64_t N2, int64_t* out);
void or_op_conv(const or_config* cfg, const int64_t* x, int64_t rows, int64_t N,
                const int64_t* g, int64_t T, int32_t correlate, int64_t* out);
/* threads of or_op_gemm's outer loop (results independent of the count) */
void or_set_threads(int32_t n);
int32_t or_max_threads(void);
void or_op_gemm(const or_config* cfg, const int64_t* A, int64_t rows_total, int64_t K,
                const int64_t* B, int64_t cols, int64_t* C);
void or_op_permute(const int64_t* x, int64_t rows, int64_t N, const int64_t* perm,
                   int64_t* out);

/* a4 + a5 at one position: Eqs. 16-19 (with the DESIGN.md readings R1-R4) and
 * Eq. 20/21.  delta[M] in, dhat[M] out (low w bits).  delta[r] is read only by
 * the check; pass check = 0 to skip it (a6 recovery).  Returns the flag. */
int32_t or_disentangle_one(const or_config* cfg, const int64_t* delta, int32_t r,
                           int64_t* dhat, int32_t check);
/* a4 + a5 over N positions, SoA M x N.  flags (nullable) gets 0/1 per position.
 * Returns the number of flagged positions. */
int64_t or_disentangle_check(const or_config* cfg, const int64_t* delta, int64_t N,
                             int32_t r, int64_t* dhat, uint8_t* flags);
/* a6: Props 1/3.  delta = M row pointers with delta[r] == NULL (absent). */
int32_t or_recover(const or_config* cfg, const int64_t* const* delta, int64_t N,
                   int32_t r, int64_t* dhat);

/* ABFT single-checksum baseline (Eqs. 3-6), w-bit arithmetic:
 * encode r_n = sum_m c_{m,n} (Eq. 4); check flags n where sum_m d_{m,n} != e_n
 * (Eq. 6), returns the count; recover d_r = e - sum_{m != r} d_m ("subtracting
 * the results of all the remaining output streams"). */
void or_abft_encode(const or_config* cfg, const int64_t* c, int64_t N, int64_t* r_out);
int64_t or_abft_check(const or_config* cfg, const int64_t* d, const int64_t* e, int64_t N, uint8_t* flags);
int32_t or_abft_recover(const or_config* cfg, const int64_t* const* d, const int64_t* e, int64_t N, int32_t r,
                        int64_t* d_r);

/* worst-case output bound of one op: op 0 scale (|s|), 1 add
 * (operand max), 2 inner/conv/gemm (operand l1 norm), 3 permute. */
int64_t or_certify(int32_t op, int64_t in_bound, int64_t operand);

/* generator wrappers (gen/ne_gen.h) for the tests. */
void or_gen_uniform(uint64_t seed, uint32_t tag, uint32_t stream, int64_t lo, int64_t hi,
                    int64_t offset, int64_t count, int64_t* out);
void or_gen_perm(uint64_t seed, uint32_t tag, int64_t n, int64_t offset, int64_t count,
                 int64_t* out);

/* test-only exhaustive loops (oracle/or_selftest.c) */
int64_t or_selftest_roundtrip_box(const or_config* cfg, int64_t H, int64_t* checked);
int64_t or_selftest_word_sweep(const or_config* cfg, const int64_t* c, int64_t* missed,
                               int64_t* silent);

#ifdef __cplusplus
}
#endif
#endif
