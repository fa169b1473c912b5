// Throughput of the forward's per-row stick math (batched_row over 64 columns) with
// 2 vs 4 warps per SMSP for the same total work per SM (tuning aid: is the math
// latency-bound at two warps per SMSP?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_17980_b200/csrc tools/ubench/ub_rowmath.cu -o tools/ubench/ub_rowmath
#include <cstdio>
#include "sb_common.cuh"
using namespace sb;

__global__ void __launch_bounds__(512) rows(float* out, int rows_per_thread, float seed) {
  float s[64];
  for (int c = 0; c < 64; ++c) s[c] = seed * (c - 32) * 0.05f + threadIdx.x * 1e-4f;
  uint32_t acc = 0;
  float a2 = 0.0f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < rows_per_thread; ++it) {
    float v[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) v[c] = s[c] + a2 * 1e-3f;
    uint32_t pk[32];
    float Q = ex2(a2), Dhi, Dlo;
    batched_row<false>(v, pk, 1.4426950408889634f * 0.125f, 64, Q, Dhi, Dlo);
#pragma unroll
    for (int c = 0; c < 32; ++c) acc += pk[c];
    a2 -= (lg2(Dhi) + lg2(Dlo)) * 1e-6f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a2 + acc;
  if (threadIdx.x == 0) out[gridDim.x * 512 + blockIdx.x] = (float)(t1 - t0);
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 512 * 4 + 148 * 4);
  const int total_rows_per_sm = 256 * 64;  // rows of 64 columns per SM
  for (int warps : {4, 8, 12, 16}) {
    const int thr = warps * 32;
    const int rpt = total_rows_per_sm / thr;
    rows<<<148, thr>>>(d, rpt, 1.0f);
    rows<<<148, thr>>>(d, rpt, 1.0f);
    cudaDeviceSynchronize();
    float c;
    cudaMemcpy(&c, d + 148 * 512, 4, cudaMemcpyDeviceToHost);
    // per SMSP: rows/4 rows of 64 elements; MUFU floor = 64 ex2 x 32 lanes / 4 per clk per row-warp
    const double rows_smsp = total_rows_per_sm / 4.0;
    printf("warps/CTA %2d (%d per SMSP): %.0f clk, %.1f clk per 32-row warp-tile-row set, MUFU floor %.1f\n",
           warps, warps / 4, c, c / (rows_smsp / 32.0), 64.0 * 32 / 4);
  }
  return 0;
}
