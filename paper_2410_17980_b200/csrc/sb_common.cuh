// Shared definitions for the stick-breaking attention kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "sm100.cuh"

namespace sb {

constexpr int kBlock = 64;     // reference d_block (blocked.py:41): skip / M / N granularity
// The forward's state array and the backward's M snapshot array start with a
// 64-float header holding the persistent kernels' work-queue counters (state[0]:
// forward; M[0]: phase 1, M[1]: phase 2), zeroed by the launcher before each
// kernel; the per-row values / tile snapshots follow.
constexpr int kSchedHeader = 64;
constexpr int kTileM = 128;    // query rows per CTA tile = two 64-row skip groups
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
// numerics.py:19: softplus switches to the identity above z = 15 (log2 units here)
constexpr float kSoftplusThr2 = 15.0f * kLog2e;

// Problem geometry shared by all kernels. Uniform batches: every (b, h) unit is
// an independent L x d problem.
struct Geom {
  int B, H, L, nb;          // nb = ceil(L / 64) key/query blocks (L = max length if varlen)
  int n_qt;                 // ceil(L / 128) query tiles
  int64_t n_tiles;          // nb*(nb+1)/2 lower-triangular 64x64 tiles per unit
  float scale_log2;         // softmax-free logit scale times log2(e)
  int64_t sb, sh, sl;       // element strides of q/k/v/o/do/dq/dk/dv (last dim contiguous)
  const int32_t* cu;        // varlen: [B+1] sequence offsets into the packed token axis
  int ugroup;               // units per grouped_order group (host: L2 working-set budget)
};

// One (sequence, head) unit: its length and where its rows, snapshots and
// per-row outputs live.  Uniform batches: unit = b*H + h, [B,H,L] layouts.
// Packed variable-length batches (cu != null): sequence b
// is tokens cu[b] .. cu[b+1]-1 of a (total, H, d) tensor, blocks restart at
// every sequence start (each sequence is an independent problem, as the
// reference runs each one separately); M/N/first_kb are packed sequence-major
// then head-major, log_rem / row_offset are (total, H).
struct Unit {
  int L, nb, n_qt;
  int64_t n_tiles;
  int trow0, tb;               // TMA coordinates: row offset and batch index
  int64_t m_off, fkb_off;      // element offsets into M / N and first_kb
  int64_t rem_off, rem_stride; // log_rem / row_offset element of row r: rem_off + r*rem_stride
  int64_t out_off;             // element offset of row 0 in q/k/v/o/do/dq/dk/dv
  int64_t z_off;               // first dZ tile of the unit in the tile workspace (ztile)
};

// dZ tile workspace (store mode of the backward): phase 1 writes every 128-row x
// 64-key dZ tile it computes, phase 2 reads them instead of recomputing dZ.  Per
// unit, tile (qt, kb) for kb < 2*qt + 2 sits at z_off + ztile(qt, kb); 16 KB each
// (the 128B-swizzled smem image, as the MMA reads it).
__device__ __forceinline__ int64_t ztile(int qt, int kb) { return (int64_t)qt * (qt + 1) + kb; }
constexpr int kZTileBytes = kTileM * kBlock * 2;

__device__ __forceinline__ Unit make_unit(const Geom& g, int b, int h) {
  Unit u;
  if (!g.cu) {
    const int64_t unit = (int64_t)b * g.H + h;
    u.L = g.L;
    u.nb = g.nb;
    u.n_qt = g.n_qt;
    u.n_tiles = g.n_tiles;
    u.trow0 = 0;
    u.tb = b;
    u.m_off = kSchedHeader + unit * g.n_tiles * kBlock;
    u.fkb_off = unit * g.nb;
    u.rem_off = unit * g.L;
    u.rem_stride = 1;
    u.out_off = (int64_t)b * g.sb + (int64_t)h * g.sh;
    u.z_off = unit * g.n_qt * (g.n_qt + 1);
  } else {
    int64_t tiles_before = 0, nb_before = 0, z_before = 0;
    for (int i = 0; i < b; ++i) {
      const int Li = g.cu[i + 1] - g.cu[i];
      const int nbi = (Li + kBlock - 1) / kBlock, nqi = (Li + kTileM - 1) / kTileM;
      tiles_before += (int64_t)nbi * (nbi + 1) / 2;
      nb_before += nbi;
      z_before += (int64_t)nqi * (nqi + 1);
    }
    const int s0 = g.cu[b];
    u.L = g.cu[b + 1] - s0;
    u.nb = (u.L + kBlock - 1) / kBlock;
    u.n_qt = (u.L + kTileM - 1) / kTileM;
    u.n_tiles = (int64_t)u.nb * (u.nb + 1) / 2;
    u.trow0 = s0;
    u.tb = 0;
    u.m_off = kSchedHeader + (tiles_before * g.H + (int64_t)h * u.n_tiles) * kBlock;
    u.fkb_off = nb_before * g.H + (int64_t)h * u.nb;
    u.rem_off = (int64_t)s0 * g.H + h;
    u.rem_stride = g.H;
    u.out_off = (int64_t)s0 * g.sl + (int64_t)h * g.sh;
    u.z_off = z_before * g.H + (int64_t)h * u.n_qt * (u.n_qt + 1);
  }
  return u;
}

// CTA -> (work item, unit): the CTAs of a group of g.ugroup units run together
// so that the K/V (or Q/dO) stream each CTA reads is shared by its neighbours in
// L2 (a unit's inputs are re-read by every CTA of that unit); inside a group
// item 0 (the heaviest, longest-processing-time first) goes first.  The host
// sizes groups to a fixed L2 budget (sb_api.cu), so a small problem (few units:
// strong scaling, short varlen batches) is one group in global LPT order.
__device__ __forceinline__ void grouped_order(int cta, int n_items, int BH, int ugroup, int& item,
                                              int& unit) {
  const int grp = cta / (ugroup * n_items);
  const int rem = cta - grp * ugroup * n_items;
  const int gsz = min(ugroup, BH - grp * ugroup);
  item = rem / gsz;
  unit = grp * ugroup + rem % gsz;
}

// Dynamic work queue of the persistent kernels: the producer warp takes item
// indices from a global counter (atomicAdd; items are independent, so results
// do not depend on which CTA runs an item) and hands them to the CTA's other
// warps through a 4-deep smem ring.  Index -1 ends the CTA's loop.
struct SchedRing {
  int* slot;       // [4] item indices
  uint64_t* full;  // [4] count 1
  uint64_t* empty; // [4] count = consumer warps
};
__device__ __forceinline__ void sched_init(const SchedRing& q, int consumers) {
  for (int i = 0; i < 4; ++i) {
    mbar_init(q.full + i, 1);
    mbar_init(q.empty + i, consumers);
  }
}
// producer warp, k-th item (whole warp; returns the index to every lane).  With
// ctr == nullptr (a forward without the M array, whose header holds the counter)
// the items are dealt statically: CTA c takes c, c + grid, c + 2 grid, ...
// The slot is handed over by the mbarriers (arrive = release, wait = acquire); its
// accesses are shared-memory atomics all the same, which compute-sanitizer's
// racecheck (unaware of mbarrier ordering for plain st/ld.shared) does not flag.
__device__ __forceinline__ int sched_produce(const SchedRing& q, int k, unsigned* ctr, int n_items) {
  int idx = 0;
  if ((threadIdx.x & 31) == 0) {
    idx = ctr ? (int)atomicAdd(ctr, 1u) : (int)(blockIdx.x + (unsigned)k * gridDim.x);
    if (idx >= n_items) idx = -1;
    if (k >= 4) mbar_wait(q.empty + (k & 3), ((k >> 2) - 1) & 1);
    atomicExch(q.slot + (k & 3), idx);
    mbar_arrive(q.full + (k & 3));
  }
  return __shfl_sync(0xffffffffu, idx, 0);
}
// consumer warp, k-th item
__device__ __forceinline__ int sched_consume(const SchedRing& q, int k) {
  mbar_wait_warp(q.full + (k & 3), (k >> 2) & 1);  // every consumer is a whole warp
  int idx = 0;
  if ((threadIdx.x & 31) == 0) {
    idx = atomicAdd(q.slot + (k & 3), 0);
    mbar_arrive(q.empty + (k & 3));
  }
  return __shfl_sync(0xffffffffu, idx, 0);
}

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

// Product-form tile math (SURVEY.md §7 "in-tile product form"): with t = e^z and
// r = 1/(1+t) = exp(lt), sigma = t*r and the suffix product of r replaces the
// suffix sum of lt, so A_c = sigma_c * prod_{c'>c} r_c' * e^a costs one ex2 and
// one rcp per element; row totals of lt come from one lg2 of the product per
// group of columns (exact slow path if that product underflows).
constexpr float kProdFloor = 7.52316384526264e-37f;  // 2^-120: lg2 of a normal product is exact enough

// Batched-reciprocal product form for one row of a 64-column tile (forward).
// Within a group of 16 columns, with P_i = prod_{k<=i} (1+t_k):
//   A_i = sigma_i * Q * prod_{k>i} r_k = t_i * Q * P_{i-1} / P_15,
// so the group needs ONE rcp (1/P_15) and a running product F = Q/P_15 * P_{i-1}
// (one FFMA per element) instead of one rcp per element.  Groups run right to
// left carrying Q (e^a times the product of r to the right).  On exit pk holds
// A packed to bf16, Q the carry past column 0, and Dhi * Dlo the tile's product
// of (1+t) (so the row total of lt is -(lg2 Dhi + lg2 Dlo) in log2 units).
// Returns false when a group product reached 2^64 (large logits): the caller
// then recomputes that row with the per-element form; values are garbage then.
// s[] is overwritten with t (the caller reloads S for the slow path).
// Masked columns (c >= lim, diagonal tiles only) get t = 0: A = 0, r = 1.
constexpr float kBatchedMax = 1.8446744073709552e19f;  // 2^64
// Wider range, tried only on a row that failed the 2^64 check (large logits), in
// the rare slow branch so the common path is unchanged: the batched form stays
// exact while every group product is < 2^126 (its rcp is normal) and the smallest
// group seed (carry / product) does not underflow, or the carried mass is
// negligible (below 2^-100 every A of the row is too).
constexpr float kBatchedWide = 8.507059173023462e37f;  // 2^126
constexpr float kSeedMin = 2.350988701644575e-38f;     // 2^-125
constexpr float kMassNeg = 7.888609052210118e-31f;     // 2^-100
__device__ __forceinline__ bool batched_seed_ok(float seed_min, float q_in) {
  return seed_min >= kSeedMin || q_in < kMassNeg;
}

// f32x2 step of pass 2 on the group pair (g, g+1) = columns (c, c+16), (c+1, c+17):
// A_i = t_i * F, F *= (1 + t_i) for two columns of both groups.
__device__ __forceinline__ float2 x2_pass2_step(const float* s, uint32_t* pk, int c, float2 F) {
  const float2 t0 = make_float2(s[c], s[c + 16]);
  const float2 t1 = make_float2(s[c + 1], s[c + 17]);
  const float2 a0 = mul2(t0, F);
  F = fma2(F, t0, F);
  const float2 a1 = mul2(t1, F);
  F = fma2(F, t1, F);
  pk[c >> 1] = pack_bf16(a0.x, a1.x);
  pk[(c + 16) >> 1] = pack_bf16(a0.y, a1.y);
  return F;
}

// The row's log2 prod (1+t) over a tile from batched_row<kDiag, true>'s Em, accurate
// for the skip decisions (blocked.py:175-176): e = prod (1+t) - 1 per group carries no
// 1 + t rounding (which for t ~ e^-8 would cost ~1e-4 of each softplus); log1p2_x2
// per group pair.  The skip-on forward evaluates it after releasing S; with the e
// chain one FMA-pipe op per element and one lg2 per group, where the exact
// per-element softplus costs a MUFU lg2 per element.
__device__ __forceinline__ float2 log1p2_x2(float2 e, float2 P);
__device__ __forceinline__ float lt_row_from_em(const float2* Em) {
  const float2 one = make_float2(1.0f, 1.0f);
  const float2 l0 = log1p2_x2(Em[0], add2(Em[0], one)), l1 = log1p2_x2(Em[1], add2(Em[1], one));
  return (l0.x + l0.y) + (l1.x + l1.y);
}

// log2(1 + e) for two groups (e >= 0: a group's prod (1+t) - 1, P = 1 + e): the
// series below 1/16, where lg2.approx of P would carry an absolute error comparable
// to the value, else lg2(P).  Branch-free (a warp-uniform branch around the lg2
// measured slower), the series on both lanes at once.
__device__ __forceinline__ float2 log1p2_x2(float2 e, float2 P) {
  const auto f2 = [](float v) { return make_float2(v, v); };
  float2 p = fma2(e, f2(-1.0f / 6.0f), f2(1.0f / 5.0f));
  p = fma2(p, e, f2(-1.0f / 4.0f));
  p = fma2(p, e, f2(1.0f / 3.0f));
  p = fma2(p, e, f2(-1.0f / 2.0f));
  p = fma2(p, e, f2(1.0f));
  const float2 small = mul2(p, mul2(e, f2(kLog2e)));
  const float b0 = lg2(P.x), b1 = lg2(P.y);
  return make_float2(e.x < 0.0625f ? small.x : b0, e.y < 0.0625f ? small.y : b1);
}

// kEm (the skip-on forward): also Em = per group prod (1+t) - 1, carried as
// e_i = e_{i-1} + t_i P_{i-1} next to the P chain (for lt_row_from_em: no 1 + t
// rounding; the product only needs relative accuracy).
template <bool kDiag, bool kEm = false>
__device__ __forceinline__ bool batched_row(float* s, uint32_t* pk, float scale_log2, int lim,
                                            float& Q, float& Dhi, float& Dlo,
                                            float2* Em = nullptr) {
#ifdef SB_NOMATH  // tuning ablation: pipeline without the stick math
#pragma unroll
  for (int c = 0; c < kBlock; c += 2) pk[c >> 1] = pack_bf16(s[c] * Q, s[c + 1] * Q);
  Dhi = Dlo = 1.0f;
  if (kEm) Em[0] = Em[1] = make_float2(0.0f, 0.0f);
  return true;
#endif
  // pass 1: t into s[], then the group products (two f32x2 chains of group pairs)
  const float2 sl2 = make_float2(scale_log2, scale_log2);
#pragma unroll
  for (int c = 0; c < kBlock; c += 2) {
    const float2 z = mul2(make_float2(s[c], s[c + 1]), sl2);
    float t0 = ex2(z.x), t1 = ex2(z.y);  // t = inf makes P = inf: slow path
    if (kDiag) {
      t0 = c < lim ? t0 : 0.0f;
      t1 = c + 1 < lim ? t1 : 0.0f;
    }
    s[c] = t0;
    s[c + 1] = t1;
  }
  float2 P[2] = {make_float2(1.0f, 1.0f), make_float2(1.0f, 1.0f)};
  if (kEm) Em[0] = Em[1] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 t2 = make_float2(s[32 * h + i], s[32 * h + 16 + i]);
      // e_i = e_{i-1} + t_i P_{i-1} (= P_i - 1 without forming 1 + t): one FFMA2
      if (kEm) Em[h] = fma2(t2, P[h], Em[h]);
      P[h] = fma2(P[h], t2, P[h]);
    }
  // group seeds F_g = Q_g / P_g, right to left
  float2 F[2];
  F[1].y = Q * rcp(P[1].y);
  F[1].x = F[1].y * rcp(P[1].x);
  F[0].y = F[1].x * rcp(P[0].y);
  F[0].x = F[0].y * rcp(P[0].x);
  Q = F[0].x;
  // pass 2: A_i = t_i * F, F *= (1 + t_i)
#pragma unroll
  for (int i = 0; i < 16; i += 2)
#pragma unroll
    for (int h = 0; h < 2; ++h) F[h] = x2_pass2_step(s, pk, 32 * h + i, F[h]);
  Dhi = P[1].y * P[1].x;
  Dlo = P[0].y * P[0].x;
  return P[0].x < kBatchedMax && P[0].y < kBatchedMax && P[1].x < kBatchedMax &&
         P[1].y < kBatchedMax;
}

// batched_row in the wider range (slow branch of the skip-off forward): s[] = raw S
// on entry.  On success pk holds A and lsum the row's log2 product of (1+t).
template <bool kDiag>
__device__ __forceinline__ bool batched_row_wide(float* s, uint32_t* pk, float scale_log2, int lim,
                                                 float Q, float& lsum) {
  constexpr int NG = kBlock / 16;
  const float q_in = Q;
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
  for (int g = 0; g < NG; ++g) ok = ok && (P[g] < kBatchedWide);
  float F[NG];
#pragma unroll
  for (int g = NG - 1; g >= 0; --g) {
    F[g] = Q * rcp(P[g]);
    Q = F[g];
  }
  if (!(ok && batched_seed_ok(Q, q_in))) return false;
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
  lsum = (lg2(P[3]) + lg2(P[2])) + (lg2(P[1]) + lg2(P[0]));
  return true;
}

}  // namespace sb
