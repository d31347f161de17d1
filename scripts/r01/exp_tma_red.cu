// Does the TMA bulk tensor reduce-add work on an INT64 tensor map (the GEMM's
// output map: box {16, 32}, 128B swizzle)?  Two reduce-adds of the same box
// into a pre-filled global tile, values chosen to carry across 32 bits and to
// wrap mod 2^64; checked on the host.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace ne::tc;

__global__ void k(const __grid_constant__ CUtensorMap m, const int64_t* src) {
  __shared__ __align__(1024) unsigned char box[4096];
  const int lane = threadIdx.x;
  for (int k = 0; k < 8; ++k) {  // row `lane`, 16-byte chunk k at k ^ (lane & 7)
    const int64_t a = src[lane * 16 + 2 * k], b = src[lane * 16 + 2 * k + 1];
    *reinterpret_cast<longlong2*>(box + lane * 128 + ((k ^ (lane & 7)) * 16)) = make_longlong2(a, b);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    for (int rep = 0; rep < 2; ++rep) {
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
                   :: "l"(reinterpret_cast<uint64_t>(&m)), "r"(16), "r"(32), "r"(smem_u32(box)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int rows = 64, cols = 32;
  std::vector<int64_t> g(rows * cols), s(32 * 16);
  for (int i = 0; i < rows * cols; ++i) g[i] = (int64_t)(0x7ffffffff0000000ull + (uint64_t)i * 0x123456789ull);
  for (int i = 0; i < 32 * 16; ++i) s[i] = (int64_t)(i % 3 == 0 ? -1 : 1) * ((int64_t)i << 33) + i;
  int64_t *dg, *ds;
  cudaMalloc(&dg, g.size() * 8);
  cudaMalloc(&ds, s.size() * 8);
  cudaMemcpy(dg, g.data(), g.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s.data(), s.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap m;
  {  // the output map of make_out_map, but UINT64 (add.u64 = add mod 2^64 for int64 too)
    EncodeTiledFn fn = encode_fn();
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 8};
    cuuint32_t box[2] = {16, 32};
    cuuint32_t estr[2] = {1, 1};
    if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, dg, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) { printf("map failed\n"); return 1; }
  }
  k<<<1, 32>>>(m, ds);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<int64_t> out(g.size());
  cudaMemcpy(out.data(), dg, g.size() * 8, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      uint64_t want = (uint64_t)g[r * cols + c];
      if (r >= 32 && c >= 16) want += 2 * (uint64_t)s[(r - 32) * 16 + (c - 16)];
      if ((uint64_t)out[r * cols + c] != want) ++bad;
    }
  printf("mismatches: %ld of %d\n", bad, rows * cols);
  return bad != 0;
}
