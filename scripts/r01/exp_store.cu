// Per-SM store throughput microbenchmark: st.global.v4 (coalesced) vs 1-D
// bulk copies smem -> global (cp.async.bulk), `ctas` CTAs each writing
// `per` bytes to its own region.  Debug tool for the GEMM epilogue drain.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_stg(int4* out, size_t per16, int reps) {
  int4* o = out + blockIdx.x * per16;
  int4 v = make_int4(threadIdx.x, 1, 2, 3);
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < per16; i += blockDim.x) o[i] = v;
}

__global__ void k_bulk(char* out, size_t per, int reps, int chunk) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) sm[i] = (char)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  char* o = out + blockIdx.x * per;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) {
    for (int r = 0; r < reps; ++r)
      for (size_t off = (size_t)w * chunk; off < per; off += (size_t)nw * chunk) {
        uint32_t s = (uint32_t)__cvta_generic_to_shared(sm + (w * chunk) % 32768);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o + off), "r"(s), "r"(chunk)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const size_t per = 256 << 10;
  char* out;
  cudaMalloc(&out, 148 * per);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  const int reps = 20;
  for (int ctas : {1, 8, 74, 148}) {
    for (int kind = 0; kind < 4; ++kind) {
      auto run = [&]() {
        if (kind == 0) k_stg<<<ctas, 256>>>((int4*)out, per / 16, reps);
        else if (kind == 1) k_stg<<<ctas, 512>>>((int4*)out, per / 16, reps);
        else if (kind == 2) k_bulk<<<ctas, 256, 32768>>>(out, per, reps, 4096);
        else k_bulk<<<ctas, 512, 32768>>>(out, per, reps, 2048);
      };
      run();
      cudaEventRecord(a);
      run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double us_per_256k = ms * 1e3 / reps;
      printf("ctas=%3d kind=%s: %.2f us per 256 KB per CTA, %.1f GB/s per SM, %.0f GB/s total\n", ctas,
             kind == 0 ? "stg256" : kind == 1 ? "stg512" : kind == 2 ? "bulk4K" : "bulk2K", us_per_256k,
             per / us_per_256k / 1e3, ctas * per / us_per_256k / 1e3);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
