// Microbenchmarks of the tcgen05 resources the stick-breaking kernels lean on
// (tuning aid, not part of the library): TMEM load bandwidth, SS-MMA throughput
// for the tile shapes used (K-major and MN-major operands), and both together.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_17980_b200/csrc \
//        tools/ubench/ub_tc.cu -o tools/ubench/ub_tc -lcuda
#include <cstdio>
#include <vector>
#include "sm100.cuh"
using namespace sb;

constexpr int ITER = 256;

// mode 0: TMEM loads only (nld warps); 1: MMA only; 2: MMA + TMEM loads
// mma_kind: 0 = 128x64 K-major (S), 1 = 128x64 MN-major A/B (dV^T), 2 = 128x128 K-major, 3 = 128x256
// ...; 8 = 128x64 TS (A from TMEM columns 256.., B K-major: phase 1's and the forward's S),
// 9 = 128x128 TS
__global__ void __launch_bounds__(544, 1) ub(int mode, int mma_kind, int nld, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 160 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 160 * 1024 + 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = *slot;
  unsigned long long t0 = clock64();
  __syncthreads();
  if (warp == 16) {
    if (lane == 0 && mode >= 1) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
      // kinds 0-3: one accumulator; 4: N=64 over 4 accumulators; 5: N=128 over 2; 6: N=256 over 2
      const int N = (mma_kind == 2 || mma_kind == 5 || mma_kind == 7 || mma_kind == 9) ? 128
                    : (mma_kind == 3 || mma_kind == 6) ? 256 : 64;
      const bool ts = mma_kind >= 8;
      const bool mn = mma_kind == 1 || mma_kind == 7;
      const int nacc = mma_kind == 4 ? 4 : (mma_kind >= 5 ? 2 : 1);
      const uint32_t idesc = idesc_bf16(128, N, mn, mn);
      uint64_t ad[8], bd[8];
      for (int k = 0; k < 8; ++k) {
        ad[k] = mn ? sdesc_sw128(a + k * 2048, 16384, 1024) : sdesc_sw128(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
        bd[k] = mn ? sdesc_sw128(b + k * 2048, N > 64 ? 16384 : 16, 1024)
                   : sdesc_sw128(b + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024);
      }
      const uint32_t cstep = mma_kind == 6 ? 256 : N;
      for (int it = 0; it < ITER; ++it) {
        const uint32_t d = tb + (it % nacc) * cstep;
        if (ts) {
#pragma unroll
          for (int k = 0; k < 8; ++k) umma_ts_at(d, tb + 256 + k * 8, bd[0], 0, idesc, 1);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) umma_ss(d, ad[k], bd[k], idesc, 1);
        }
      }
      umma_commit(bar);
      mbar_wait(bar, 0);
      out[blockIdx.x * 2 + 0] = clock64() - t0;
    }
  } else if (warp < nld && mode == 3) {
    // generic-proxy smem stores (16 B per thread) into 96..160 KB, concurrent with the MMAs
    uint32_t base = smem_u32(smem + 96 * 1024) + (warp * 32 + lane) * 16;
    for (int it = 0; it < ITER * 4; ++it)
      st_shared_v4(base + (it & 7) * 8192, it, it + 1, it + 2, it + 3);
    if (lane == 0 && warp == 0) out[blockIdx.x * 2 + 1] = clock64() - t0;
  } else if (warp < nld && mode != 1) {
    // loads from columns 256..511 (disjoint from the MMA accumulator at 0..255)
    const uint32_t ta = tb + 256 + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64 % 256;
    float v[64];
    float acc = 0.f;
    for (int it = 0; it < ITER; ++it) {
      tmem_ld32(ta, v);
      tmem_ld32(ta + 32, v + 32);
      tmem_wait_ld();
      acc += v[it & 63];
    }
    if (acc == 12345.f) out[0] = 1;
    if (lane == 0 && warp == 0) out[blockIdx.x * 2 + 1] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 2 * 8);
  cudaFuncSetAttribute(ub, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const char* kn[] = {"128x64 K-major", "128x64 MN-major", "128x128 K-major", "128x256 K-major",
                      "128x64 4 acc", "128x128 2 acc", "128x256 2 acc", "128x128 MN/MN",
                      "128x64 TS", "128x128 TS"};
  const int Ns[] = {64, 64, 128, 256, 64, 128, 256, 128, 64, 128};
  std::vector<unsigned long long> h(296);
  auto run = [&](int mode, int kind, int nld) {
    cudaMemset(d, 0, 296 * 8);
    ub<<<148, 544, 170 * 1024>>>(mode, kind, nld, d);
    ub<<<148, 544, 170 * 1024>>>(mode, kind, nld, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(h.data(), d, 296 * 8, cudaMemcpyDeviceToHost);
    double m = 0, l = 0;
    for (int i = 0; i < 148; ++i) { m += h[2 * i]; l += h[2 * i + 1]; }
    m /= 148; l /= 148;
    if (mode >= 1) {
      double flop = 2.0 * 128 * Ns[kind] * 16 * 8 * ITER;
      printf("mode %d %-16s nld %2d: MMA %8.0f clk  = %6.1f clk per K=16 MMA, %6.0f FLOP/clk/SM", mode, kn[kind], nld,
             m, m / (8 * ITER), flop / m);
    }
    if (mode == 3) {
      double bytes = (double)nld * 32 * 16 * ITER * 4;
      printf(" | STS (warp 0) %8.0f clk = %6.1f B/clk/SM", l, bytes / l);
    } else if (mode != 1) {
      double bytes = (double)nld * 32 * 64 * 4 * ITER;
      printf("%s TMEM ld (warp 0) %8.0f clk = %6.1f B/clk/SM", mode >= 1 ? " |" : "mode 0 ", l, bytes / l);
    }
    printf("\n");
  };
  for (int nld : {4, 8, 16}) run(0, 0, nld);
  for (int k = 0; k < 10; ++k) run(1, k, 0);
  for (int nld : {4, 8}) run(2, 0, nld);
  run(2, 1, 8);
  for (int nld : {4, 8, 16}) run(3, 2, nld);
  for (int nld : {4, 8, 16}) run(3, 0, nld);
  return 0;
}
