// C4 gather floor on B200: random aligned chunks of 32, 64, 128 and 256 bytes
// from an 8 GiB buffer (the C4 AoS eps: 2^28 positions x 32 B), the same
// number of accesses for every chunk size, plus cache-hint variants of the
// 32-byte access.  Timed with CUDA events (no profiler) and, separately,
// profiled with ncu for dram__sectors_read / lts__t_sectors_* (DRAM bytes
// fetched per access vs bytes used).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o c4_floor c4_floor.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_fill(uint64_t* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = mix(i ^ 0x5555);
}

// V: 0 = ld.global.nc.L1::no_allocate (C4's form), 1 = + .L2::evict_first, 2 = default ld.global,
//    3 = ld.global.cs (streaming), 4 = .L2::evict_last
template <int BYTES, int V>
__global__ void __launch_bounds__(256) k_gather(const uint64_t* __restrict__ x, int64_t nchunks, int64_t nacc,
                                                uint64_t seed, uint64_t* __restrict__ out) {
  uint64_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int U = 8;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < nacc; i0 += stride * U) {
    const uint64_t* p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      const int64_t c = (int64_t)(mix(seed + (uint64_t)(i < nacc ? i : 0)) % (uint64_t)nchunks);
      p[u] = x + c * (BYTES / 8);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u * stride >= nacc) break;
#pragma unroll
      for (int b = 0; b < BYTES / 32; ++b) {
        uint64_t a0, a1, a2, a3;
        const uint64_t* q = p[u] + 4 * b;
        if (V == 0)
          asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                       : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(q));
        else if (V == 1)
          asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
                       : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(q));
        else if (V == 2)
          asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(q));
        else if (V == 3)
          asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(q));
        else
          asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v4.u64 {%0,%1,%2,%3}, [%4];"
                       : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(q));
        acc ^= a0 + a1 + a2 + a3;
      }
    }
  }
  out[blockIdx.x * (int64_t)blockDim.x + threadIdx.x] = acc;
}

template <int BYTES, int V>
static void run(const char* name, const uint64_t* x, int64_t nbytes, int64_t nacc, uint64_t* out, int grid) {
  const int64_t nchunks = nbytes / BYTES;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_gather<BYTES, V><<<grid, 256>>>(x, nchunks, nacc, 1, out);  // warm
  cudaEventRecord(e0);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) k_gather<BYTES, V><<<grid, 256>>>(x, nchunks, nacc, 7 + r, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double acc_per_s = nacc / (ms * 1e-3);
  printf("%-28s bytes/access %4d  accesses %lld  %8.3f ms  %7.2f G access/s  used %7.1f GB/s  at 128 B/access %7.1f GB/s\n",
         name, BYTES, (long long)nacc, ms, acc_per_s / 1e9, acc_per_s * BYTES / 1e9, acc_per_s * 128 / 1e9);
}

int main(int argc, char** argv) {
  const int64_t nbytes = 8ll << 30;  // 8 GiB: the C4 AoS eps (2^28 x 32 B)
  const int64_t nacc = 1ll << 28;    // C4's number of gathered positions
  const bool profile = argc > 1;     // one launch each (for ncu)
  uint64_t *x, *out;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * 32;
  cudaMalloc(&x, nbytes);
  cudaMalloc(&out, (size_t)grid * 256 * 8);
  k_fill<<<nsm * 8, 256>>>(x, nbytes / 8);
  cudaDeviceSynchronize();
  if (profile) {
    k_gather<32, 0><<<grid, 256>>>(x, nbytes / 32, nacc, 7, out);
    k_gather<64, 0><<<grid, 256>>>(x, nbytes / 64, nacc, 7, out);
    k_gather<128, 0><<<grid, 256>>>(x, nbytes / 128, nacc, 7, out);
    k_gather<256, 0><<<grid, 256>>>(x, nbytes / 256, nacc / 2, 7, out);
    k_gather<32, 1><<<grid, 256>>>(x, nbytes / 32, nacc, 7, out);
    k_gather<32, 2><<<grid, 256>>>(x, nbytes / 32, nacc, 7, out);
    k_gather<32, 3><<<grid, 256>>>(x, nbytes / 32, nacc, 7, out);
    k_gather<32, 4><<<grid, 256>>>(x, nbytes / 32, nacc, 7, out);
    cudaDeviceSynchronize();
    return 0;
  }
  run<32, 0>("32B nc.no_allocate", x, nbytes, nacc, out, grid);
  run<64, 0>("64B nc.no_allocate", x, nbytes, nacc, out, grid);
  run<128, 0>("128B nc.no_allocate", x, nbytes, nacc, out, grid);
  run<256, 0>("256B nc.no_allocate", x, nbytes, nacc / 2, out, grid);
  run<32, 1>("32B L2::evict_first", x, nbytes, nacc, out, grid);
  run<32, 2>("32B default", x, nbytes, nacc, out, grid);
  run<32, 3>("32B .cs", x, nbytes, nacc, out, grid);
  run<32, 4>("32B L2::evict_last", x, nbytes, nacc, out, grid);
  // cudaLimitMaxL2FetchGranularity = 32 (the smallest the driver takes)
  if (cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32) == cudaSuccess) {
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("cudaLimitMaxL2FetchGranularity -> %zu\n", v);
    run<32, 0>("32B nc, L2 fetch limit 32", x, nbytes, nacc, out, grid);
  }
  printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
