// Throughput of the forward's per-row stick math (batched_row over 64 columns) with
// 2 vs 4 warps per SMSP for the same total work per SM (tuning aid: is the math
// latency-bound at two warps per SMSP?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_17980_b200/csrc tools/ubench/ub_rowmath.cu -o tools/ubench/ub_rowmath
#include <cstdio>
#include <cstring>
#include "sb_common.cuh"
using namespace sb;

// The scalar form batched_row had before the f32x2 rewrite (same operations per
// element): the f32x2 version must reproduce it bit for bit.
template <bool kDiag>
__device__ __forceinline__ bool batched_row_scalar(float* s, uint32_t* pk, float scale_log2, int lim,
                                                   float& Q, float& Dhi, float& Dlo) {
  constexpr int NG = kBlock / 16;
  float P[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) P[g] = 1.0f;
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const int c = 16 * g + i;
      float tt = ex2(s[c] * scale_log2);
      if (kDiag) tt = c < lim ? tt : 0.0f;
      s[c] = tt;
      P[g] = fmaf(P[g], tt, P[g]);
    }
  bool ok = true;
#pragma unroll
  for (int g = 0; g < NG; ++g) ok = ok && (P[g] < kBatchedMax);
  float F[NG];
#pragma unroll
  for (int g = NG - 1; g >= 0; --g) {
    F[g] = Q * rcp(P[g]);
    Q = F[g];
  }
#pragma unroll
  for (int i = 0; i < 16; i += 2)
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const int c = 16 * g + i;
      const float a0 = s[c] * F[g];
      F[g] = fmaf(F[g], s[c], F[g]);
      const float a1 = s[c + 1] * F[g];
      F[g] = fmaf(F[g], s[c + 1], F[g]);
      pk[c >> 1] = pack_bf16(a0, a1);
    }
  Dhi = P[3] * P[2];
  Dlo = P[1] * P[0];
  return ok;
}

template <int kX2>
__global__ void __launch_bounds__(512) rows(float* out, int rows_per_thread, float seed, float scale) {
  __shared__ float4 sm[4][512];
  float s[64];
  for (int c = 0; c < 64; ++c) s[c] = seed * (c - 32) * 0.05f + threadIdx.x * 1e-4f;
  uint32_t acc = 0;
  float a2 = 0.0f;
  for (int j = 0; j < 4; ++j) sm[j][threadIdx.x] = make_float4(s[4 * j], s[4 * j + 1], s[4 * j + 2], s[4 * j + 3]);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < rows_per_thread; ++it) {
    // the S row arrives like a TMEM load: straight into registers, no FMA-pipe work
    float v[64];
#pragma unroll
    for (int c = 0; c < 64; c += 4) {
      const float4 x = sm[(c / 4 + it) & 3][threadIdx.x];
      // distinct per column and iteration (one ALU-pipe LOP3 each, no FMA-pipe work)
      const int m = (it + c) & 63;
      v[c] = __int_as_float(__float_as_int(x.x) ^ m);
      v[c + 1] = __int_as_float(__float_as_int(x.y) ^ (m + 1));
      v[c + 2] = __int_as_float(__float_as_int(x.z) ^ (m + 2));
      v[c + 3] = __int_as_float(__float_as_int(x.w) ^ (m + 3));
    }
    uint32_t pk[32];
    float Q = ex2(a2), Dhi, Dlo;
    if (kX2)
      batched_row<false>(v, pk, scale, 64, Q, Dhi, Dlo);
    else
      batched_row_scalar<false>(v, pk, scale, 64, Q, Dhi, Dlo);
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
  float* h = new float[148 * 512];
  float* keep = new float[4 * 148 * 512];
  for (int x2 = 0; x2 < 2; ++x2)
  for (int warps : {4, 8, 12, 16}) {
    const int thr = warps * 32;
    const int rpt = total_rows_per_sm / thr;
    auto kern = x2 ? rows<1> : rows<0>;
    kern<<<148, thr>>>(d, rpt, 1.0f, 1.4426950408889634f * 0.0883883476f);
    kern<<<148, thr>>>(d, rpt, 1.0f, 1.4426950408889634f * 0.0883883476f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 148 * thr * 4, cudaMemcpyDeviceToHost);
    float* ref = keep + (warps / 4 - 1) * 148 * 512;
    if (!x2) memcpy(ref, h, 148 * thr * 4);  // the f32x2 pass must reproduce it bit for bit
    else if (memcmp(h, ref, 148 * thr * 4) != 0) printf("MISMATCH f32x2 vs scalar\n");
    printf("%s ", x2 ? "f32x2 " : "scalar");
    float c;
    cudaMemcpy(&c, d + 148 * 512, 4, cudaMemcpyDeviceToHost);
    // per SMSP: rows/4 rows of 64 elements; MUFU floor = 64 ex2 x 32 lanes / 4 per clk per row-warp
    const double rows_smsp = total_rows_per_sm / 4.0;
    printf("warps/CTA %2d (%d per SMSP): %.0f clk, %.1f clk per 32-row warp-tile-row set, MUFU floor %.1f\n",
           warps, warps / 4, c, c / (rows_smsp / 32.0), 64.0 * 32 / 4);
  }
  return 0;
}
