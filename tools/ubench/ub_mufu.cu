// MUFU.EX2 rate reachable by ONE warp per SMSP (the phase-1 ping-pong runs one
// recompute warp per SMSP at a time), with and without part of the ex2 moved to
// a polynomial on the FMA pipe (tuning aid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_17980_b200/csrc tools/ubench/ub_mufu.cu -o tools/ubench/ub_mufu
#include <cstdio>
#include "sm100.cuh"
using namespace sb;
constexpr int IT = 2048;

// 2^x for x in [-127, 64] on the FMA pipe: x = j + f (j = floor), 2^f by a degree-5
// minimax-style polynomial, exponent added as an integer.  Two lanes at a time.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -127.0f);
  x.y = fmaxf(x.y, -127.0f);
  const float2 j = make_float2(floorf(x.x), floorf(x.y));
  const float2 f = add2(x, make_float2(-j.x, -j.y));
  float2 p = make_float2(1.8775767e-3f, 1.8775767e-3f);
  p = fma2(p, f, make_float2(8.9893397e-3f, 8.9893397e-3f));
  p = fma2(p, f, make_float2(5.5826318e-2f, 5.5826318e-2f));
  p = fma2(p, f, make_float2(2.4015361e-1f, 2.4015361e-1f));
  p = fma2(p, f, make_float2(6.9315308e-1f, 6.9315308e-1f));
  p = fma2(p, f, make_float2(1.0f, 1.0f));
  const int jx = (int)j.x, jy = (int)j.y;
  return make_float2(__int_as_float(__float_as_int(p.x) + (jx << 23)),
                     __int_as_float(__float_as_int(p.y) + (jy << 23)));
}

// OP 0: all MUFU; OP 1: every third column pair on the FMA pipe; OP 2: one in two; OP 3: all poly
template <int OP>
__global__ void __launch_bounds__(256) k(float* out, float seed) {
  float a[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) a[i] = -0.001f * (threadIdx.x + i) + seed;
  const float2 sc = make_float2(-0.9f, -0.9f);
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int c = 0; c < 64; c += 2) {
      const float2 z = mul2(make_float2(a[c], a[c + 1]), sc);
      const bool poly = OP == 3 || (OP == 1 && (c % 6) == 4) || (OP == 2 && (c % 4) == 2);
      if (poly) {
        const float2 t = ex2_poly2(z);
        a[c] = t.x;
        a[c + 1] = t.y;
      } else {
        a[c] = ex2(z.x);
        a[c + 1] = ex2(z.y);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = (float)(t1 - t0);
}

template <int OP>
void run(const char* name, float* d, int nthr) {
  k<OP><<<148, nthr>>>(d, 0.1f);
  k<OP><<<148, nthr>>>(d, 0.1f);
  cudaDeviceSynchronize();
  float c;
  cudaMemcpy(&c, d + 148 * nthr, 4, cudaMemcpyDeviceToHost);
  const double elems = (double)IT * 64;  // per thread
  printf("%-18s %3d thr (%d warp/SMSP): %8.0f clk, %.2f clk per 64-element row per warp, "
         "%.1f elem/clk/SM\n", name, nthr, nthr / 128, c, c / IT, elems * nthr / c);
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 1024 * 4 + 4096);
  for (int n : {128, 256}) {
    run<0>("mufu", d, n);
    run<1>("1/3 poly", d, n);
    run<2>("1/2 poly", d, n);
    run<3>("all poly", d, n);
  }
  return 0;
}
