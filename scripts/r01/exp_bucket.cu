// Experiment: bucketed permutation + blocked inner product (C4 shape) vs the
// direct random gather.  M = 4 AoS int64 positions (one 32-B sector each),
// n = 2^28, blocks of 1024, pi a bijection.  Because pi is a bijection, the
// sources falling in window k (2^S positions) are exactly 2^S, so bucket k is
// the fixed entry range [k 2^S, (k+1) 2^S) — no histogram pass.
//   pass A: e = (i << 32) | pi(i) written into bucket pi(i) >> S (cursor per bucket)
//   pass B: walk entries in order (one L2-resident window at a time), gather
//           x[pi(i)] from L2, red.add x * v[i & 1023] into out[i >> 10] (8 MB, L2)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp_bucket exp_bucket.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__host__ __device__ inline uint32_t perm28(uint32_t x) {  // a bijection of [0, 2^28)
  const uint32_t MASK = (1u << 28) - 1;
  for (int r = 0; r < 3; ++r) {
    x = (x * 0x9E3779Bu + 0x7F4A7C1u + r) & MASK;  // odd multiplier: bijective mod 2^28
    x ^= x >> 13;
    x = (x * 0x5BD1E99u) & MASK | 0;
    x ^= x >> 11;
  }
  return x & MASK;
}

__global__ void k_init(int64_t* x, int32_t* pi, int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    pi[i] = (int32_t)perm28((uint32_t)i);
    for (int m = 0; m < 4; ++m) x[i * 4 + m] = (int64_t)((i * 2654435761ull + m * 97) % 100003) - 50000;
    if (i < 1024) v[i] = (int32_t)(i * 37 % 8191) - 4096;
  }
}

__global__ void __launch_bounds__(256) k_direct(const int64_t* __restrict__ x, const int32_t* __restrict__ pi,
                                                const int32_t* __restrict__ v, int64_t n, int64_t* __restrict__ out) {
  // one warp per block of 1024: 32 positions per lane
  const int lane = threadIdx.x & 31;
  const int64_t nb = n >> 10;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; b < nb;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t a[4] = {0, 0, 0, 0};
#pragma unroll 8
    for (int u = 0; u < 32; ++u) {
      const int64_t i = (b << 10) + u * 32 + lane;
      const int64_t s = __ldcs(pi + i);
      int64_t q0, q1, q2, q3;
      asm volatile("ld.global.nc.L1::no_allocate.v4.s64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(q0), "=l"(q1), "=l"(q2), "=l"(q3) : "l"(x + s * 4));
      const int64_t vv = v[u * 32 + lane];
      a[0] += q0 * vv; a[1] += q1 * vv; a[2] += q2 * vv; a[3] += q3 * vv;
    }
#pragma unroll
    for (int m = 0; m < 4; ++m)
      for (int o = 16; o; o >>= 1) a[m] += __shfl_xor_sync(0xffffffffu, a[m], o);
    if (lane < 4) out[b * 4 + lane] = a[lane];
  }
}

template <int S>
__global__ void __launch_bounds__(256) k_bucket(const int32_t* __restrict__ pi, int64_t n,
                                                unsigned long long* __restrict__ cursor, uint64_t* __restrict__ ent) {
  // each CTA: 256 threads x 16 entries; smem per-bucket counts, one global atomic per (CTA, bucket)
  constexpr int NBMAX = 1024;
  __shared__ uint32_t cnt[NBMAX];
  __shared__ unsigned long long base[NBMAX];
  const int nbk = (int)(n >> S);
  for (int64_t c0 = (int64_t)blockIdx.x * 4096; c0 < n; c0 += (int64_t)gridDim.x * 4096) {
    for (int k = threadIdx.x; k < nbk; k += 256) cnt[k] = 0;
    __syncthreads();
    uint32_t s[16], slot[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      s[u] = (uint32_t)__ldcs(pi + c0 + u * 256 + threadIdx.x);
      slot[u] = atomicAdd(&cnt[s[u] >> S], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nbk; k += 256)
      base[k] = cnt[k] ? atomicAdd(&cursor[k], (unsigned long long)cnt[k]) : 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint64_t i = (uint64_t)(c0 + u * 256 + threadIdx.x);
      const uint32_t k = s[u] >> S;
      ent[((uint64_t)k << S) + base[k] + slot[u]] = (i << 32) | s[u];
    }
    __syncthreads();
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_apply(const int64_t* __restrict__ x, const uint64_t* __restrict__ ent,
                                               const int32_t* __restrict__ v, int64_t n, int64_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t q = __ldcs(ent + e);
    const uint32_t i = (uint32_t)(q >> 32), s = (uint32_t)q;
    int64_t q0, q1, q2, q3;
    asm volatile("ld.global.v4.s64 {%0,%1,%2,%3}, [%4];" : "=l"(q0), "=l"(q1), "=l"(q2), "=l"(q3) : "l"(x + (int64_t)s * 4));
    const int64_t vv = __ldg(v + (i & 1023));
    unsigned long long* o = reinterpret_cast<unsigned long long*>(out + (int64_t)(i >> 10) * 4);
    if (MODE == 0) {
      atomicAdd(o + 0, (unsigned long long)(q0 * vv));
      atomicAdd(o + 1, (unsigned long long)(q1 * vv));
      atomicAdd(o + 2, (unsigned long long)(q2 * vv));
      atomicAdd(o + 3, (unsigned long long)(q3 * vv));
    } else {  // red (no return)
      asm volatile("red.global.add.u64 [%0], %1;" ::"l"(o + 0), "l"(q0 * vv) : "memory");
      asm volatile("red.global.add.u64 [%0], %1;" ::"l"(o + 1), "l"(q1 * vv) : "memory");
      asm volatile("red.global.add.u64 [%0], %1;" ::"l"(o + 2), "l"(q2 * vv) : "memory");
      asm volatile("red.global.add.u64 [%0], %1;" ::"l"(o + 3), "l"(q3 * vv) : "memory");
    }
  }
}

// atomics alone: 2^30 red.add into 8 MB at random (hashed) block indices
__global__ void __launch_bounds__(256) k_atom_only(int64_t n, int64_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = perm28((uint32_t)e) >> 10;
    unsigned long long* o = reinterpret_cast<unsigned long long*>(out + (int64_t)b * 4);
#pragma unroll
    for (int m = 0; m < 4; ++m) asm volatile("red.global.add.u64 [%0], %1;" ::"l"(o + m), "l"(e) : "memory");
  }
}

int main(int argc, char** argv) {
  const int64_t n = 1ll << 28;
  int64_t* x; int32_t* pi; int32_t* v; int64_t *o1, *o2; uint64_t* ent; unsigned long long* cur;
  CK(cudaMalloc(&x, n * 32)); CK(cudaMalloc(&pi, n * 4)); CK(cudaMalloc(&v, 4096));
  CK(cudaMalloc(&o1, (n >> 10) * 32)); CK(cudaMalloc(&o2, (n >> 10) * 32));
  CK(cudaMalloc(&ent, n * 8)); CK(cudaMalloc(&cur, 8 * 1024));
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  k_init<<<nsm * 8, 256>>>(x, pi, v, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  auto T = [&](const char* name, auto fn, double bytes) {
    fn(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-28s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  T("direct gather", [&] { k_direct<<<nsm * 8, 256>>>(x, pi, v, n, o1); }, n * 36.0);
  T("atomics only 2^30", [&] { cudaMemsetAsync(o2, 0, (n >> 10) * 32); k_atom_only<<<nsm * 8, 256>>>(n, o2); }, n * 32.0);
  for (int S : {20, 21, 22}) {
    auto bucket = [&] {
      cudaMemsetAsync(cur, 0, 8 * 1024);
      if (S == 20) k_bucket<20><<<nsm * 4, 256>>>(pi, n, cur, ent);
      if (S == 21) k_bucket<21><<<nsm * 4, 256>>>(pi, n, cur, ent);
      if (S == 22) k_bucket<22><<<nsm * 4, 256>>>(pi, n, cur, ent);
    };
    char nm[64];
    snprintf(nm, 64, "bucket pass S=%d", S);
    T(nm, bucket, n * 12.0);
    T("apply (atomicAdd)", [&] { cudaMemsetAsync(o2, 0, (n >> 10) * 32); k_apply<0><<<nsm * 8, 256>>>(x, ent, v, n, o2); }, n * 40.0);
    T("apply (red)", [&] { cudaMemsetAsync(o2, 0, (n >> 10) * 32); k_apply<1><<<nsm * 8, 256>>>(x, ent, v, n, o2); }, n * 40.0);
    int64_t* h1 = (int64_t*)malloc((n >> 10) * 32);
    int64_t* h2 = (int64_t*)malloc((n >> 10) * 32);
    CK(cudaMemcpy(h1, o1, (n >> 10) * 32, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2, o2, (n >> 10) * 32, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t i = 0; i < (n >> 10) * 4; ++i) bad += h1[i] != h2[i];
    printf("  mismatches vs direct: %lld\n", (long long)bad);
    free(h1); free(h2);
  }
  return 0;
}
