// Shared-memory 128-bit store patterns (tuning aid): the row-per-lane 128B-swizzle
// store of the stick warps (lane L writes chunk k ^ (L & 7) of row L) vs a linear
// pattern (lane L writes bytes 16L..16L+15 of a 512-byte run).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_17980_b200/csrc tools/ubench/ub_sts.cu -o tools/ubench/ub_sts
#include <cstdio>
#include "sm100.cuh"
using namespace sb;
constexpr int IT = 2048;

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out) {
  __shared__ __align__(1024) uint8_t buf[8][4096];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = smem_u32(buf[warp]);
  uint32_t v = lane;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t a;
      if (MODE == 0) a = base + lane * 128 + ((c ^ (lane & 7)) << 4);  // row per lane, swizzled
      else a = base + c * 512 + lane * 16;                               // linear
      st_shared_v4(a, v, v + 1, v + 2, v + 3);
      v += 7;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (float)(t1 - t0);
  if (v == 12345) out[1000] = 1.f;
}

int main() {
  float* d;
  cudaMalloc(&d, 4096 * 4);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, 256>>>(d); else k<1><<<148, 256>>>(d);
    }
    cudaDeviceSynchronize();
    float c;
    cudaMemcpy(&c, d, 4, cudaMemcpyDeviceToHost);
    // 8 warps x IT x 8 stores of 512 B; smem bandwidth 128 B/clk -> ideal 4 clk per store
    printf("%s: %.2f clk per warp-store (ideal 4 at 128 B/clk)\n", mode ? "linear" : "row-swizzled",
           c / (8.0 * IT * 8));
  }
  return 0;
}
