/*
 * or_selftest.c — exhaustive loops used by the oracle's own pins
 * (tests/test_oracle_exhaustive.py).  TEST INFRASTRUCTURE ONLY.
 *
 * They only compose the oracle's public functions (entangle, disentangle,
 * check); they live in C because the loops run 10^7-10^9 times.
 */
#include "ne_oracle.h"

/* Brute force over EVERY input triple... tuple in [-H, H]^M (M = 3 only: the
 * box is H^3) and every excluded stream r: disentangle(entangle(c), r) == c.
 * Entangled values are wrapped to the w-bit container (or_entangle does).
 * Returns the number of failing (tuple, r) pairs; *checked gets the count. */
int64_t or_selftest_roundtrip_box(const or_config* cfg, int64_t H, int64_t* checked) {
  int64_t fails = 0, n = 0;
  if (cfg->M != 3) return -1;
  int64_t c[3], eps[3], d[3];
  for (c[0] = -H; c[0] <= H; ++c[0])
    for (c[1] = -H; c[1] <= H; ++c[1])
      for (c[2] = -H; c[2] <= H; ++c[2]) {
        or_entangle(cfg, c, 1, eps);
        for (int32_t r = 0; r < 3; ++r) {
          int32_t f = or_disentangle_one(cfg, eps, r, d, 1);
          ++n;
          if (f || d[0] != c[0] || d[1] != c[1] || d[2] != c[2]) ++fails;
        }
      }
  if (checked) *checked = n;
  return fails;
}

/* Single-word corruption sweep at one position (w <= 20 only): entangle the
 * M-tuple c, then for every stream s and every w-bit value v != eps_s
 * substitute v for delta_s and run disentangle + check excluding r = 0.
 * missed = corruptions the check does not flag; silent = missed ones whose
 * disentangled outputs differ from c (undetected wrong results).
 * Returns the number of corruptions tried. */
int64_t or_selftest_word_sweep(const or_config* cfg, const int64_t* c, int64_t* missed,
                               int64_t* silent) {
  const int32_t M = cfg->M, w = cfg->w;
  if (w > 20 || M > 64) return -1;
  int64_t eps[64], delta[64], d[64], tried = 0, miss = 0, sil = 0;
  or_entangle(cfg, c, 1, eps);
  const int64_t lo = -((int64_t)1 << (w - 1)), hi = ((int64_t)1 << (w - 1)) - 1;
  for (int32_t s = 0; s < M; ++s) {
    for (int64_t v = lo; v <= hi; ++v) {
      if (v == eps[s]) continue;
      for (int32_t m = 0; m < M; ++m) delta[m] = eps[m];
      delta[s] = v;
      ++tried;
      int32_t f = or_disentangle_one(cfg, delta, 0, d, 1);
      if (!f) {
        ++miss;
        for (int32_t m = 0; m < M; ++m)
          if (d[m] != c[m]) {
            ++sil;
            break;
          }
      }
    }
  }
  *missed = miss;
  *silent = sil;
  return tried;
}
