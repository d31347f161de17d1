/*
 * ne_gendev.h — device-side fill of the seeded synthetic inputs (libne.so).
 *
 * Test/bench infrastructure: the same counter-based generator as
 * gen/ne_gen.h (the one module the oracle and the CUDA path share), run on
 * the GPU so that 2^28-element streams are created in place.  These calls
 * hold none of the method's arithmetic.  Same conventions as ne.h: device
 * pointers owned by the caller, asynchronous on `stream`.
 */
#ifndef NE_GENDEV_H
#define NE_GENDEV_H

#include <stdint.h>

#include "ne.h"

#ifdef __cplusplus
extern "C" {
#endif

/* out[i] = uniform[lo, hi) of counter (seed, tag, gstream, offset + i), int32.
 * Errors: NE_EINVAL if hi - lo is not in (0, 2^32] or the values overflow int32. */
ne_status ne_gen_uniform_i32(uint64_t seed, uint32_t tag, uint32_t gstream, int64_t lo,
                             int64_t hi, int64_t offset, int64_t count, int32_t* out,
                             ne_stream_t stream);

/* out[i] = perm(seed, tag, n, i) for i < n: the seeded Feistel bijection. */
ne_status ne_gen_perm_i32(uint64_t seed, uint32_t tag, int64_t n, int32_t* out,
                          ne_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
