/*
 * ne_gen.h — seeded, counter-based synthetic input generator.
 *
 * This is the ONE module shared by the oracle (oracle/) and the CUDA path
 * (paper_1604_04740_b200/csrc/).  It holds none of the method's arithmetic
 * (no entanglement, no LSB op, no disentanglement): it only maps a counter
 * (seed, tag, stream, index) to a pseudo-random integer, and an index to a
 * seeded bijection of [0, n).  Both sides include it; neither side includes
 * the other.
 *
 * Why it exists: the paper draws its streams from unspecified integer
 * distributions (§V, lines 1085-1121 name none), so the inputs are
 * ours by definition.  Counter-based generation
 * lets the GPU fill 2^28-element streams in place and the oracle recompute any
 * single element on demand, bit for bit.
 *
 * Definitions (DESIGN.md §"Input recipe"):
 *   mix(z)        = splitmix64 finaliser of (z + 0x9E3779B97F4A7C15)
 *   u(s,t,m,i)    = mix( mix(s ^ (t << 40) ^ (m << 32)) + i )
 *   uniform[lo,hi)= lo + (int64)( ((u >> 32) * (uint64)(hi - lo)) >> 32 )
 *                   (valid for 0 < hi - lo <= 2^32)
 *   perm(s,t,n,i) = cycle-walking 4-round balanced Feistel bijection of
 *                   [0, 2^b) restricted to [0, n), b = even bit width with
 *                   2^b >= n, round function mix(key_r ^ R) & mask.
 *
 * Tags: 1 = streams c, 2 = second addend set, 3 = conv taps, 4 = GEMM A,
 *       5 = GEMM B, 6 = permutation, 7 = inner-product vector,
 *       8 = outer-product vector, 9 = fault masks.
 */
#ifndef NE_GEN_H
#define NE_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define NE_GEN_FN static __host__ __device__ __forceinline__
#else
#define NE_GEN_FN static inline
#endif

#define NE_TAG_C      1u
#define NE_TAG_ADDEND 2u
#define NE_TAG_TAPS   3u
#define NE_TAG_GEMM_A 4u
#define NE_TAG_GEMM_B 5u
#define NE_TAG_PERM   6u
#define NE_TAG_VEC    7u
#define NE_TAG_OUTER  8u
#define NE_TAG_FAULT  9u

NE_GEN_FN uint64_t ne_gen_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

NE_GEN_FN uint64_t ne_gen_key(uint64_t seed, uint32_t tag, uint32_t stream) {
  return ne_gen_mix(seed ^ ((uint64_t)tag << 40) ^ ((uint64_t)stream << 32));
}

NE_GEN_FN uint64_t ne_gen_u64(uint64_t key, uint64_t idx) {
  return ne_gen_mix(key + idx);
}

/* uniform integer in [lo, hi), 0 < hi - lo <= 2^32 */
NE_GEN_FN int64_t ne_gen_uniform(uint64_t key, uint64_t idx, int64_t lo, int64_t hi) {
  uint64_t u = ne_gen_u64(key, idx);
  uint64_t span = (uint64_t)(hi - lo);
  return lo + (int64_t)(((u >> 32) * span) >> 32);
}

/* even bit width b >= 2 with 2^b >= n */
NE_GEN_FN uint32_t ne_gen_perm_bits(uint64_t n) {
  uint32_t b = 2;
  while (b < 62 && (1ull << b) < n) b += 2;
  return b;
}

NE_GEN_FN uint64_t ne_gen_feistel(uint64_t key, uint32_t b, uint64_t x) {
  uint32_t h = b / 2;
  uint64_t mask = (1ull << h) - 1ull;
  uint64_t L = x >> h, R = x & mask;
  for (uint32_t r = 0; r < 4; ++r) {
    uint64_t F = ne_gen_mix(key ^ ((uint64_t)r << 56) ^ R) & mask;
    uint64_t nL = R;
    R = L ^ F;
    L = nL;
  }
  return (L << h) | R;
}

/* seeded bijection of [0, n): perm(i), by cycle walking (n >= 1, i < n) */
NE_GEN_FN uint64_t ne_gen_perm(uint64_t key, uint64_t n, uint64_t i) {
  uint32_t b = ne_gen_perm_bits(n);
  uint64_t x = ne_gen_feistel(key, b, i);
  while (x >= n) x = ne_gen_feistel(key, b, x);
  return x;
}

#endif /* NE_GEN_H */
