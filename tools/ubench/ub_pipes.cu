// Per-SM throughput of the instructions the stick math uses (tuning aid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_17980_b200/csrc tools/ubench/ub_pipes.cu -o tools/ubench/ub_pipes
#include <cstdio>
#include "sm100.cuh"
using namespace sb;
constexpr int IT = 4096;

template <int OP>
__global__ void __launch_bounds__(512) k(float* out, float seed) {
  float a[8];
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = ex2(a[i]);
      if (OP == 1) a[i] = rcp(a[i]);
      if (OP == 2) a[i] = fmaf(a[i], 1.0001f, 0.5f);
      if (OP == 3) a[i] = a[i] * 1.0001f;
      if (OP == 4) { acc += pack_bf16(a[i], a[(i + 1) & 7]); a[i] = __uint_as_float(acc); }
      if (OP == 5) a[i] = lg2(a[i]);
      if (OP == 6) a[i] = fminf(a[i], 3.0f) + 1.0f;
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = (float)(t1 - t0);
}

template <int OP>
void run(const char* name, float* d, int nthr) {
  k<OP><<<148, nthr>>>(d, 0.1f);
  k<OP><<<148, nthr>>>(d, 0.1f);
  cudaDeviceSynchronize();
  float c;
  cudaMemcpy(&c, d + 148 * nthr, 4, cudaMemcpyDeviceToHost);
  double ops = (double)nthr * IT * 8;
  printf("%-10s %4d thr: %8.0f clk -> %6.1f ops/clk/SM\n", name, nthr, c, ops / c);
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 1024 * 4 + 4096);
  for (int n : {256, 512}) {
    run<0>("ex2", d, n);
    run<1>("rcp", d, n);
    run<5>("lg2", d, n);
    run<2>("ffma", d, n);
    run<3>("fmul", d, n);
    run<4>("f2fp+iadd", d, n);
    run<6>("fmnmx+add", d, n);
  }
  return 0;
}
