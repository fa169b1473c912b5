// Shared definitions for the stick-breaking attention kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "sm100.cuh"

namespace sb {

constexpr int kBlock = 64;     // reference d_block (blocked.py:41): skip / M / N granularity
constexpr int kTileM = 128;    // query rows per CTA tile = two 64-row skip groups
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
// numerics.py:19: softplus switches to the identity above z = 15 (log2 units here)
constexpr float kSoftplusThr2 = 15.0f * kLog2e;

// Problem geometry shared by all kernels. Uniform batches: every (b, h) unit is
// an independent L x d problem.
struct Geom {
  int B, H, L, nb;          // nb = ceil(L / 64) key/query blocks
  int n_qt;                 // ceil(L / 128) query tiles
  int64_t n_tiles;          // nb*(nb+1)/2 lower-triangular 64x64 tiles per unit
  float scale_log2;         // softmax-free logit scale times log2(e)
  int64_t sb, sh, sl;       // element strides of q/k/v/o/do/dq/dk/dv (last dim contiguous)
};

// tile(qb, kb) = qb*(qb+1)/2 + kb, the reference's (qb, kb) snapshot key order
__device__ __forceinline__ int64_t tile_index(int qb, int kb) {
  return (int64_t)qb * (qb + 1) / 2 + kb;
}

// softplus(z) * log2(e) given Z = z*log2(e) and t = e^z = 2^Z.
// numerics.py:33-47: log1p(exp(z)) for z <= 15, z otherwise. log1p is
// evaluated as a short series for t < 1/16 (lg2.approx has an absolute, not
// relative, error bound, which would swamp tiny softplus values) and with the
// MUFU lg2 of 1+t otherwise.
__device__ __forceinline__ float softplus2(float Z, float t) {
  float p = fmaf(t, -1.0f / 6.0f, 1.0f / 5.0f);
  p = fmaf(p, t, -1.0f / 4.0f);
  p = fmaf(p, t, 1.0f / 3.0f);
  p = fmaf(p, t, -1.0f / 2.0f);
  p = fmaf(p, t, 1.0f);
  const float small = p * (t * kLog2e);
  const float big = lg2(1.0f + t);
  float sp = t < 0.0625f ? small : big;
  return Z > kSoftplusThr2 ? Z : sp;
}

}  // namespace sb
