// ne_host.cu — host-side part of the C ABI: configuration (a0), certification,
// validation helpers, diag reset.  See include/ne.h for the contract.
#include <cuda_runtime.h>

#include <climits>

#include "ne_internal.cuh"

namespace ne {

static int64_t pow2i(int e) { return (int64_t)1 << e; }

ne_status validate_cfg(const ne_config* cfg) {
  if (!cfg) return NE_EINVAL;
  if (cfg->M < 3 || cfg->M > NE_MAX_M) return NE_ECONFIG;
  if (cfg->w != 64) return NE_ECONFIG;  // w = 32 containers: DESIGN.md "next"
  if (cfg->l < 1 || cfg->k < 1 || cfg->k > cfg->l) return NE_ECONFIG;
  if ((cfg->M - 1) * cfg->l + cfg->k > cfg->w) return NE_ECONFIG;  // Eq. 12
  return NE_OK;
}

// Eq. 13 and, for M = 3, Eq. 11: the smaller (R6).
int64_t range_hi(const ne_config* cfg) {
  const int l = cfg->l, k = cfg->k, M = cfg->M;
  // Eq. 13: 2^((M-3)l+k) (2^(l-1) - 1); exponent <= w - 2l - 1 + ... < 63
  __int128 e13 = (__int128)pow2i((M - 3) * l + k) * (pow2i(l - 1) - 1);
  __int128 hi = e13;
  if (M == 3) {
    __int128 e11 = (__int128)pow2i(l + k - 1) - pow2i(l);
    if (e11 < hi) hi = e11;
  }
  if (hi > (__int128)INT64_MAX) hi = INT64_MAX;
  return (int64_t)hi;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

int grid_for(int64_t work_items, int threads, int per_sm) {
  int64_t need = (work_items + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

ne_status launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NE_OK : NE_ECUDA;
}

__global__ void k_diag_reset(ne_diag* d) {
  d->range_violations = 0;
  d->first_bad = LLONG_MAX;
  d->fault_positions = 0;
  d->first_fault = LLONG_MAX;
}

}  // namespace ne

using namespace ne;

extern "C" ne_status ne_config_for(int32_t M, int32_t w, ne_config* out) {
  if (!out) return NE_EINVAL;
  if (M < 3 || M > NE_MAX_M || w < 4 || w > 64) return NE_ECONFIG;
  // Eq. 12: maximise (M-2)l + k, (M-1)l + k <= w, 1 <= k <= l.
  // For fixed l the best k is min(l, w - (M-1)l); scan l, keep ties at larger l.
  int best_v = -1, best_l = 0, best_k = 0;
  for (int l = 1; (M - 1) * l + 1 <= w; ++l) {
    int k = w - (M - 1) * l;
    if (k > l) k = l;
    if (k < 1) continue;
    int v = (M - 2) * l + k;
    if (v >= best_v) {  // '>=' : a later (larger) l wins a tie (reading R5)
      best_v = v;
      best_l = l;
      best_k = k;
    }
  }
  if (best_v < 0) return NE_ECONFIG;
  out->M = M;
  out->w = w;
  out->l = best_l;
  out->k = best_k;
  return NE_OK;
}

// a0 host calls accept both container widths (w = 32: the ne_*_w32 path)
static ne_status validate_cfg_host(const ne_config* cfg) {
  if (!cfg) return NE_EINVAL;
  if (cfg->w == 32) {
    if (cfg->M < 3 || cfg->M > NE_MAX_M || cfg->l < 1 || cfg->k < 1 || cfg->k > cfg->l ||
        (cfg->M - 1) * cfg->l + cfg->k > 32)
      return NE_ECONFIG;
    return NE_OK;
  }
  return validate_cfg(cfg);
}

extern "C" ne_status ne_dynamic_range(const ne_config* cfg, int64_t* hi) {
  ne_status st = validate_cfg_host(cfg);
  if (st != NE_OK) return st;
  if (!hi) return NE_EINVAL;
  *hi = range_hi(cfg);
  return NE_OK;
}

extern "C" ne_status ne_certify(const ne_config* cfg, ne_op_kind op, int64_t in_bound,
                                int64_t operand, int64_t* out_bound) {
  ne_status st = validate_cfg_host(cfg);
  if (st != NE_OK) return st;
  if (!out_bound || in_bound < 0 || operand < 0) return NE_EINVAL;
  __int128 b;
  switch (op) {
    case NE_OP_SCALE: b = (__int128)in_bound * operand; break;
    case NE_OP_ADD: b = (__int128)in_bound + operand; break;
    case NE_OP_LINEAR: b = (__int128)in_bound * operand; break;
    case NE_OP_PERMUTE: b = in_bound; break;
    default: return NE_EINVAL;
  }
  *out_bound = b > (__int128)INT64_MAX ? INT64_MAX : (int64_t)b;
  return b <= (__int128)range_hi(cfg) ? NE_OK : NE_ERANGE;
}

extern "C" int32_t ne_gemm_limbs_for(const ne_config* cfg, int64_t in_bound) {
  if (validate_cfg(cfg) != NE_OK || in_bound < 0) return -1;
  // |eps| <= (2^l + 1) in_bound; L balanced base-256 digits cover
  // |x| <= 127 * (256^L - 1) / 255 (all digits at +-127 / -128 side).
  __int128 eb = ((__int128)1 << cfg->l) * in_bound + in_bound;
  for (int L = 1; L <= 8; ++L) {
    __int128 cap = 0, p = 1;
    for (int i = 0; i < L; ++i) {
      cap += 127 * p;
      p *= 256;
    }
    if (eb <= cap) return L;
  }
  return 8;
}

// Cheapest exact digit plan for the tensor-core GEMM operand:
// an entangled value c_m + 2^l c_{m-1} with |c| <= 127 and l >= 8 is exactly
// two int8 digits in base 2^l; otherwise balanced base-256 digits.
extern "C" int32_t ne_gemm_limb_plan(const ne_config* cfg, int64_t in_bound, int32_t* limb_bits) {
  if (validate_cfg(cfg) != NE_OK || in_bound < 0 || !limb_bits) return -1;
  const int32_t L8 = ne_gemm_limbs_for(cfg, in_bound);
  if (in_bound <= 127 && cfg->l >= 8 && cfg->l <= 63 && L8 > 2) {
    *limb_bits = cfg->l;
    return 2;
  }
  *limb_bits = 8;
  return L8;
}

extern "C" ne_status ne_diag_reset(ne_diag* diag, ne_stream_t stream) {
  if (!diag) return NE_EINVAL;
  k_diag_reset<<<1, 1, 0, cs(stream)>>>(diag);
  return launch_status();
}
