// Microbenchmark: random 32-byte gathers (one AoS position of M = 4 int64)
// with different load flavours, to find one that does not over-fetch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_idx(int32_t* idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    idx[i] = (int32_t)(mix(i) % (uint64_t)n);
}

template <int V>
__device__ __forceinline__ void ld32(const int64_t* p, int64_t (&o)[4]) {
  if (V == 0) {  // default caching
    asm volatile("ld.global.v2.s64 {%0,%1}, [%4]; ld.global.v2.s64 {%2,%3}, [%4+16];"
                 : "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]) : "l"(p));
  } else if (V == 1) {  // non-coherent, no L1 allocate
    asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0,%1}, [%4]; ld.global.nc.L1::no_allocate.v2.s64 {%2,%3}, [%4+16];"
                 : "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]) : "l"(p));
  } else if (V == 2) {  // cache-streaming (what k_pinner used)
    asm volatile("ld.global.cs.v2.s64 {%0,%1}, [%4]; ld.global.cs.v2.s64 {%2,%3}, [%4+16];"
                 : "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]) : "l"(p));
  } else if (V == 3) {  // one 256-bit load (sm_100+)
    asm volatile("ld.global.v4.s64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]) : "l"(p));
  } else if (V == 4) {  // L1 bypass (.cg)
    asm volatile("ld.global.cg.v2.s64 {%0,%1}, [%4]; ld.global.cg.v2.s64 {%2,%3}, [%4+16];"
                 : "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]) : "l"(p));
  } else if (V == 5) {  // 256-bit, nc no_allocate
    asm volatile("ld.global.nc.L1::no_allocate.v4.s64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]) : "l"(p));
  }
}

template <int V, int U>
__global__ void __launch_bounds__(256) k_gather(const int64_t* __restrict__ x, const int32_t* __restrict__ idx,
                                                int64_t n, int64_t* __restrict__ out) {
  int64_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += stride * U) {
    int64_t j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) j[u] = (i0 + u * stride < n) ? idx[i0 + u * stride] : -1;
    int64_t v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j[u] >= 0) ld32<V>(x + j[u] * 4, v[u]);
      else v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u][0] ^ v[u][1] ^ v[u][2] ^ v[u][3];
  }
  if (acc == 0x123456789) out[0] = acc;
}

template <int V, int U>
float run(const int64_t* x, const int32_t* idx, int64_t n, int64_t* out, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gather<V, U><<<grid, 256>>>(x, idx, n, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_gather<V, U><<<grid, 256>>>(x, idx, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}


// TMA (bulk copy engine) gather: each lane copies its U positions (32 B each)
// global -> shared with cp.async.bulk, completion on one mbarrier per warp.
template <int U>
__global__ void __launch_bounds__(256) k_gather_bulk(const int64_t* __restrict__ x, const int32_t* __restrict__ idx,
                                                     int64_t n, int64_t* __restrict__ out) {
  __shared__ __align__(128) int64_t buf[8][32 * U * 4];
  __shared__ __align__(8) uint64_t bar[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp]);
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  int64_t acc = 0;
  uint32_t phase = 0;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32 * U; base < n; base += nwarps * 32 * U) {
    const int64_t cnt = (n - base) < 32 * U ? (n - base) : 32 * U;
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"((uint32_t)(cnt * 32)) : "memory");
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t p = base + u * 32 + lane;
      if (p < n) {
        int64_t j = idx[p];
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(&buf[warp][(u * 32 + lane) * 4]);
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];"
                     ::"r"(dst), "l"(x + j * 4), "r"(b) : "memory");
      }
    }
    asm volatile("{\n .reg .pred P1;\n W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W;\n}" ::"r"(b), "r"(phase) : "memory");
    phase ^= 1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t* q = &buf[warp][(u * 32 + lane) * 4];
      acc += q[0] ^ q[1] ^ q[2] ^ q[3];
    }
    __syncwarp();
  }
  if (acc == 0x123456789) out[0] = acc;
}

template <int U>
float run_bulk(const int64_t* x, const int32_t* idx, int64_t n, int64_t* out, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gather_bulk<U><<<grid, 256>>>(x, idx, n, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_gather_bulk<U><<<grid, 256>>>(x, idx, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  const int64_t n = 1ll << 28;
  int64_t* x;
  int32_t* idx;
  int64_t* out;
  cudaMalloc(&x, n * 32);
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&out, 64);
  cudaMemset(x, 1, n * 32);
  k_idx<<<148 * 8, 256>>>(idx, n);
  cudaDeviceSynchronize();
  int grids[3] = {148 * 4, 148 * 8, 148 * 32};
  const char* names[6] = {"default", "nc.no_alloc", "cs", "v4.b64(256b)", "cg", "nc v4.b64"};
  for (int g = 0; g < 3; ++g) {
    float t[6];
    t[0] = run<0, 8>(x, idx, n, out, grids[g]);
    t[1] = run<1, 8>(x, idx, n, out, grids[g]);
    t[2] = run<2, 8>(x, idx, n, out, grids[g]);
    t[3] = run<3, 8>(x, idx, n, out, grids[g]);
    t[4] = run<4, 8>(x, idx, n, out, grids[g]);
    t[5] = run<5, 8>(x, idx, n, out, grids[g]);
    for (int v = 0; v < 6; ++v)
      printf("grid %6d %-14s %7.3f ms  algorithmic %6.0f GB/s\n", grids[g], names[v], t[v], n * 36 / t[v] / 1e6);
  }
  for (int g = 0; g < 3; ++g) {
    float t4 = run_bulk<4>(x, idx, n, out, grids[g]);
    float t2 = run_bulk<2>(x, idx, n, out, grids[g]);
    printf("grid %6d bulk U=4 %7.3f ms (%6.0f GB/s)  U=2 %7.3f ms (%6.0f GB/s)\n", grids[g], t4, n * 36 / t4 / 1e6, t2, n * 36 / t2 / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
