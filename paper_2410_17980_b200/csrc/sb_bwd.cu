// Stick-breaking attention two-phase backward (K2 + K3 of SURVEY.md §2.2), sm_100a.
//
// Restates blocked_backward_twophase (reference blocked.py:299-392):
//   recompute_tile (:325-335): z, lt, A = exp(z + suffix_cumsum(lt) + M)
//   dW = dO V^T - row_offset; dAt = A*dW; sigma = 1 - exp(lt);
//   dZ = dAt - sigma*(prefix_cumsum(dAt) + b)
// Phase 1 (:337-357): per query tile, key blocks left to right from first_kb,
//   b carried in registers, N snapshot = b in effect per tile, dQ += dZ K.
// Phase 2 (:367-386): per 64-key block, query tiles top to bottom over visited
//   tiles, b = N snapshot, dK += dZ^T Q, dV += A^T dO — owned rows, no atomics,
//   deterministic.  dK^T and dV^T are accumulated in TMEM with M = head_dim
//   (A^T / dZ^T reach the tensor core through MN-major smem descriptors).
//
// Stick warps are split like the forward's: warp w owns rows 32*(w%4)..+31 and
// key columns [16*(w/4), +16) of the 64-column tile; per row, the four column
// groups exchange (1) their suffix totals of lt (A needs everything to its
// right) and (2) their prefix totals of dAt (dZ needs everything to its left)
// through shared memory, one named barrier each.
#include "sb_args.cuh"

namespace sb {

constexpr int kBwdGroups = 4;
constexpr int kBwdCG = kBlock / kBwdGroups;  // 16 key columns per stick thread
constexpr int kBwdStick = 128 * kBwdGroups;  // 512 stick threads
constexpr int kBwdThreads = kBwdStick + 64;  // + TMA producer warp + MMA warp

// Per-row, per-tile stick math shared by both phases (product form, see
// sb_common.cuh: A_c = sigma_c * prod_{c'>c} r_c' * e^M, sigma = t/(1+t)).
struct RowTile {
  float z[kBwdCG];   // Z = z*log2(e), later dAt
  float cl[kBwdCG];  // sigma_c * in-group suffix product of r, later prefix sums of dAt
  float sg[kBwdCG];  // sigma(z) = 1 - exp(lt), 0 where masked
  float w[kBwdCG];   // dW = dO.V^T
};

// pass 1: sigma, r and the in-group suffix products; returns the group's product of r.
template <bool kDiag>
__device__ __forceinline__ float bwd_pass1(RowTile& t, float scale_log2, int c0, int lim) {
  return prod_pass<kBwdCG, kDiag>(t.z, t.cl, t.sg, scale_log2, c0, lim);
}

// pass 2: A = cl*base (base = e^M * product of r right of this group),
// dAt = A*(dW - off), in-group inclusive prefix sums of dAt; A packed to bf16
// into pa (may be null). Returns the group's dAt total.
__device__ __forceinline__ float bwd_pass2(RowTile& t, float base, float off, uint32_t* pa) {
  float pfx = 0.0f;
#pragma unroll
  for (int c = 0; c < kBwdCG; c += 2) {
    const float A0 = t.cl[c] * base;
    const float A1 = t.cl[c + 1] * base;
    if (pa) pa[c >> 1] = pack_bf16(A0, A1);
    t.z[c] = A0 * (t.w[c] - off);
    t.z[c + 1] = A1 * (t.w[c + 1] - off);
    pfx += t.z[c];
    t.cl[c] = pfx;
    pfx += t.z[c + 1];
    t.cl[c + 1] = pfx;
  }
  return pfx;
}

// pass 3: dZ = dAt - sigma*(prefix(dAt) + b), b = left groups' dAt total + b in effect.
__device__ __forceinline__ void bwd_pass3(const RowTile& t, float b, uint32_t* pz) {
#pragma unroll
  for (int c = 0; c < kBwdCG; c += 2)
    pz[c >> 1] = pack_bf16(t.z[c] - t.sg[c] * (t.cl[c] + b),
                           t.z[c + 1] - t.sg[c + 1] * (t.cl[c + 1] + b));
}

// 16 columns (two 16-byte chunks) of one row of a 128B-swizzled K-major tile
__device__ __forceinline__ void store_cols_sw128(uint32_t row_addr, int r, int gi,
                                                 const uint32_t* pk) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int chunk = gi * 2 + c;
    st_shared_v4(row_addr + ((chunk ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                 pk[4 * c + 3]);
  }
}

// product of the r-products of the groups right of mine
__device__ __forceinline__ float exchange_right_prod(const float* xch, int par, int gi, int r) {
  float p = 1.0f;
#pragma unroll
  for (int g2 = 0; g2 < kBwdGroups; ++g2)
    if (g2 > gi) p *= xch[(par * kBwdGroups + g2) * 128 + r];
  return p;
}

__device__ __forceinline__ void exchange_sums(const float* xch, int par, int gi, int r,
                                              float& right, float& left, float& tot) {
  right = left = tot = 0.0f;
#pragma unroll
  for (int g2 = 0; g2 < kBwdGroups; ++g2) {
    const float v = xch[(par * kBwdGroups + g2) * 128 + r];
    tot += v;
    if (g2 > gi) right += v;
    if (g2 < gi) left += v;
  }
}

// ============================================================================
// Phase 1: dQ and N.  CTA = (b, h, 128-row query tile).
template <int D>
struct BwdQCfg {
  static constexpr int kStages = D == 128 ? 3 : 4;
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kKVBytes = kBlock * D * 2;
  static constexpr int kZBytes = kTileM * kBlock * 2;
  static constexpr int kOffQ = 0;
  static constexpr int kOffDO = kOffQ + kQBytes;
  static constexpr int kOffK = kOffDO + kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKVBytes;
  static constexpr int kOffZ = kOffV + kStages * kKVBytes;
  static constexpr int kOffX = kOffZ + 2 * kZBytes;  // 2 x [2][NG][128] f32
  static constexpr int kOffBar = kOffX + 2 * 2 * kBwdGroups * 128 * 4;
  static constexpr int kNumBars = 1 + 3 * kStages + 2 * 4 + 1;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS = 0, kColW = 128, kColQ = 256;
};

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    sb_bwd_q_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const BwdArgs args) {
  using C = BwdQCfg<D>;
  constexpr int ST = C::kStages;
  constexpr int kProdWarp = 4 * kBwdGroups, kMmaWarp = kProdWarp + 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BH = g.B * g.H;
  const int qt = g.n_qt - 1 - (int)(blockIdx.x / BH);
  const int bh = (int)(blockIdx.x % BH);
  const int b = bh / g.H, h = bh % g.H;
  const int64_t unit = (int64_t)b * g.H + h;
  const int qb0 = 2 * qt;
  const bool has1 = qb0 + 1 < g.nb;
  const int kb_hi = has1 ? qb0 + 1 : qb0;
  const int* fkb = args.first_kb + unit * g.nb;
  const int f0 = fkb[qb0];
  const int f1 = has1 ? fkb[qb0 + 1] : f0;
  const int kb_lo = min(f0, f1);
  const int n = kb_hi - kb_lo + 1;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_qdo = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_vfull = bar_kfull + ST;
  uint64_t* bar_kvempty = bar_vfull + ST;
  uint64_t* bar_sfull = bar_kvempty + ST;
  uint64_t* bar_sempty = bar_sfull + 2;
  uint64_t* bar_zfull = bar_sempty + 2;
  uint64_t* bar_zempty = bar_zfull + 2;
  uint64_t* bar_done = bar_zempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  float* xch1 = reinterpret_cast<float*>(smem + C::kOffX);
  float* xch2 = xch1 + 2 * kBwdGroups * 128;

  if (threadIdx.x == 0) {
    mbar_init(bar_qdo, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_kfull + s, 1);
      mbar_init(bar_vfull + s, 1);
      mbar_init(bar_kvempty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_sfull + s, 1);
      mbar_init(bar_sempty + s, kBwdStick);
      mbar_init(bar_zfull + s, kBwdStick);
      mbar_init(bar_zempty + s, 1);
    }
    mbar_init(bar_done, 1);
    fence_mbar_init();
  }
  if (warp == kProdWarp) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == kProdWarp) {
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_do);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      const int row0 = qt * kTileM;
      mbar_expect_tx(bar_qdo, 2 * C::kQBytes);
      for (int c = 0; c < D / 64; ++c) {
        tma_load_4d(&tm_q, bar_qdo, smem + C::kOffQ + c * (kTileM * 128), c * 64, row0, h, b);
        tma_load_4d(&tm_do, bar_qdo, smem + C::kOffDO + c * (kTileM * 128), c * 64, row0, h, b);
      }
      for (int j = 0; j < n; ++j) {
        const int s = j % ST;
        if (j >= ST) mbar_wait(bar_kvempty + s, ((j / ST) - 1) & 1);
        const int kb = kb_lo + j;
        mbar_expect_tx(bar_kfull + s, C::kKVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_k, bar_kfull + s, smem + C::kOffK + s * C::kKVBytes + c * (kBlock * 128),
                      c * 64, kb * kBlock, h, b);
        mbar_expect_tx(bar_vfull + s, C::kKVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_v, bar_vfull + s, smem + C::kOffV + s * C::kKVBytes + c * (kBlock * 128),
                      c * 64, kb * kBlock, h, b);
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T, dO V^T
      constexpr uint32_t idesc_q = idesc_bf16(128, D, 0, 1);   // dZ K: K is MN-major
      const uint32_t q_addr = smem_u32(smem + C::kOffQ);
      const uint32_t do_addr = smem_u32(smem + C::kOffDO);
      const uint32_t k_addr = smem_u32(smem + C::kOffK);
      const uint32_t v_addr = smem_u32(smem + C::kOffV);
      const uint32_t z_addr = smem_u32(smem + C::kOffZ);
      mbar_wait(bar_qdo, 0);
      auto issue_dq = [&](int i) {
        const int s = i % ST;
        mbar_wait(bar_zfull + (i & 1), (i >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kBlock / 16; ++k) {
          const uint64_t ad = sdesc_sw128(z_addr + (i & 1) * C::kZBytes + k * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(k_addr + s * C::kKVBytes + k * 2048, kBlock * 128, 1024);
          umma_ss(tbase + C::kColQ, ad, bd, idesc_q, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(bar_zempty + (i & 1));
        umma_commit(bar_kvempty + s);
      };
      for (int j = 0; j < n; ++j) {
        const int s = j % ST;
        mbar_wait(bar_kfull + s, (j / ST) & 1);
        mbar_wait(bar_vfull + s, (j / ST) & 1);
        if (j >= 2) mbar_wait(bar_sempty + (j & 1), ((j >> 1) + 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
          const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
          umma_ss(tbase + C::kColS + (j & 1) * 64, sdesc_sw128(q_addr + off, 16, 1024),
                  sdesc_sw128(k_addr + s * C::kKVBytes + offk, 16, 1024), idesc_s, k > 0);
        }
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
          const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
          umma_ss(tbase + C::kColW + (j & 1) * 64, sdesc_sw128(do_addr + off, 16, 1024),
                  sdesc_sw128(v_addr + s * C::kKVBytes + offk, 16, 1024), idesc_s, k > 0);
        }
        umma_commit(bar_sfull + (j & 1));
        if (j >= 1) issue_dq(j - 1);
      }
      issue_dq(n - 1);
      umma_commit(bar_done);
    }
  } else {
    const int quarter = warp & 3, gi = warp >> 2;
    const int r = quarter * 32 + lane;
    const int half = r >> 6;
    const int my_qb = qb0 + half;
    const int row = qt * kTileM + r;
    const bool row_valid = row < g.L;
    const bool half_exists = my_qb < g.nb;
    const int my_first = half ? f1 : f0;
    const int c0 = gi * kBwdCG;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const float off = (args.row_offset && row_valid) ? args.row_offset[unit * g.L + row] : 0.0f;
    const float* Mrow = args.M + unit * g.n_tiles * kBlock + (r & 63);
    float* Nrow = args.N + unit * g.n_tiles * kBlock + (r & 63);
    const uint32_t z_row = smem_u32(smem + C::kOffZ) + r * 128;
    float bsum = 0.0f;  // running b (blocked.py:342, :354)

    for (int j = 0; j < n; ++j) {
      const int kb = kb_lo + j;
      const int par = j & 1;
      const bool live = half_exists && row_valid && kb >= my_first && kb <= my_qb;
      const int lim = (kb == my_qb) ? (r & 63) : kBlock;
      const int64_t t = tile_index(my_qb, kb) * kBlock;
      const float Ma = live ? Mrow[t] : 0.0f;
      mbar_wait(bar_sfull + par, (j >> 1) & 1);
      tc_fence_after();
      RowTile rt;
      tmem_ld16(tbase + lane_base + C::kColS + par * 64 + c0, rt.z);
      tmem_ld16(tbase + lane_base + C::kColW + par * 64 + c0, rt.w);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar_sempty + par);

      const bool diag = kb == my_qb;  // warp-uniform
      float part = 1.0f, right, left, tot;
      if (live)
        part = diag ? bwd_pass1<true>(rt, g.scale_log2, c0, lim)
                    : bwd_pass1<false>(rt, g.scale_log2, c0, lim);
      xch1[(par * kBwdGroups + gi) * 128 + r] = part;
      named_bar_sync(1, kBwdStick);
      right = exchange_right_prod(xch1, par, gi, r);
      part = live ? bwd_pass2(rt, ex2(Ma) * right, off, nullptr) : 0.0f;
      xch2[(par * kBwdGroups + gi) * 128 + r] = part;
      named_bar_sync(1, kBwdStick);
      exchange_sums(xch2, par, gi, r, right, left, tot);
      uint32_t pz[kBwdCG / 2];
      if (live) {
        bwd_pass3(rt, left + bsum, pz);
        if (gi == 0) Nrow[t] = bsum;  // b in effect for this tile (blocked.py:353)
        bsum += tot;
      } else {
#pragma unroll
        for (int c = 0; c < kBwdCG / 2; ++c) pz[c] = 0u;
      }
      if (j >= 2) mbar_wait(bar_zempty + par, ((j >> 1) + 1) & 1);
      store_cols_sw128(z_row + par * C::kZBytes, r, gi, pz);
      fence_proxy_async_smem();
      mbar_arrive(bar_zfull + par);
    }

    mbar_wait(bar_done, 0);
    tc_fence_after();
    constexpr int DC = D / kBwdGroups;
    const float scale = g.scale_log2 * kLn2;
    float v[DC];
    if constexpr (DC == 16) {
      tmem_ld16(tbase + lane_base + C::kColQ + gi * DC, v);
    } else {
      tmem_ld32(tbase + lane_base + C::kColQ + gi * DC, v);
    }
    tmem_wait_ld();
    if (row_valid) {
      uint4* dst = reinterpret_cast<uint4*>(args.dq + (int64_t)b * g.sb + (int64_t)h * g.sh +
                                            (int64_t)row * g.sl + gi * DC);
#pragma unroll
      for (int q4 = 0; q4 < DC / 8; ++q4)
        dst[q4] = make_uint4(pack_bf16(v[8 * q4] * scale, v[8 * q4 + 1] * scale),
                             pack_bf16(v[8 * q4 + 2] * scale, v[8 * q4 + 3] * scale),
                             pack_bf16(v[8 * q4 + 4] * scale, v[8 * q4 + 5] * scale),
                             pack_bf16(v[8 * q4 + 6] * scale, v[8 * q4 + 7] * scale));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProdWarp) tmem_dealloc<C::kTmemCols>(tbase);
}

// ============================================================================
// Phase 2: dK and dV.  CTA = (b, h, 64-key block kb); query tiles stream.
template <int D>
struct BwdKVCfg {
  static constexpr int kStages = D == 128 ? 2 : 3;
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kKVBytes = kBlock * D * 2;
  static constexpr int kPBytes = kTileM * kBlock * 2;
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kKVBytes;
  static constexpr int kOffQ = kOffV + kKVBytes;                  // stage s: Q at +s*2*kQBytes
  static constexpr int kOffA = kOffQ + kStages * 2 * kQBytes;     // A (single buffer)
  static constexpr int kOffZ = kOffA + kPBytes;                   // dZ (single buffer)
  static constexpr int kOffX = kOffZ + kPBytes;
  static constexpr int kOffBar = kOffX + 2 * 2 * kBwdGroups * 128 * 4;
  static constexpr int kNumBars = 1 + 2 * kStages + 2 + 2 + 4 + 1;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS = 0, kColW = 128, kColV = 256, kColK = 320;
};

// first live query tile >= qt for key block kb (a tile (qb, kb) is live when
// the forward visited it: first_kb[qb] <= kb <= qb, blocked.py:372-373)
__device__ __forceinline__ int next_live_qt(const int* fkb, int nb, int n_qt, int kb, int qt) {
  for (; qt < n_qt; ++qt) {
    const int q0 = 2 * qt, q1 = 2 * qt + 1;
    if (q0 >= kb && fkb[q0] <= kb) return qt;
    if (q1 < nb && q1 >= kb && fkb[q1] <= kb) return qt;
  }
  return n_qt;
}

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    sb_bwd_kv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                     const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     const BwdArgs args) {
  using C = BwdKVCfg<D>;
  constexpr int ST = C::kStages;
  constexpr int kProdWarp = 4 * kBwdGroups, kMmaWarp = kProdWarp + 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BH = g.B * g.H;
  const int kb = (int)(blockIdx.x / BH);  // small kb first: they own the longest columns
  const int bh = (int)(blockIdx.x % BH);
  const int b = bh / g.H, h = bh % g.H;
  const int64_t unit = (int64_t)b * g.H + h;
  const int* fkb = args.first_kb + unit * g.nb;
  const int qt_first = next_live_qt(fkb, g.nb, g.n_qt, kb, kb >> 1);

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_kv = bars;
  uint64_t* bar_qfull = bars + 1;
  uint64_t* bar_qempty = bar_qfull + ST;
  uint64_t* bar_sfull = bar_qempty + ST;
  uint64_t* bar_sempty = bar_sfull + 2;
  uint64_t* bar_afull = bar_sempty + 2;
  uint64_t* bar_aempty = bar_afull + 1;
  uint64_t* bar_zfull = bar_aempty + 1;
  uint64_t* bar_zempty = bar_zfull + 1;
  uint64_t* bar_done = bar_zempty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  float* xch1 = reinterpret_cast<float*>(smem + C::kOffX);
  float* xch2 = xch1 + 2 * kBwdGroups * 128;

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_qfull + s, 1);
      mbar_init(bar_qempty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_sfull + s, 1);
      mbar_init(bar_sempty + s, kBwdStick);
    }
    mbar_init(bar_afull, kBwdStick);
    mbar_init(bar_aempty, 1);
    mbar_init(bar_zfull, kBwdStick);
    mbar_init(bar_zempty, 1);
    mbar_init(bar_done, 1);
    fence_mbar_init();
  }
  if (warp == kProdWarp) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const bool any = qt_first < g.n_qt;

  if (warp == kProdWarp) {
    if (lane == 0 && any) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_do);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      mbar_expect_tx(bar_kv, 2 * C::kKVBytes);
      for (int c = 0; c < D / 64; ++c) {
        tma_load_4d(&tm_k, bar_kv, smem + C::kOffK + c * (kBlock * 128), c * 64, kb * kBlock, h, b);
        tma_load_4d(&tm_v, bar_kv, smem + C::kOffV + c * (kBlock * 128), c * 64, kb * kBlock, h, b);
      }
      int j = 0;
      for (int qt = qt_first; qt < g.n_qt; qt = next_live_qt(fkb, g.nb, g.n_qt, kb, qt + 1), ++j) {
        const int s = j % ST;
        if (j >= ST) mbar_wait(bar_qempty + s, ((j / ST) - 1) & 1);
        uint8_t* qdst = smem + C::kOffQ + s * 2 * C::kQBytes;
        mbar_expect_tx(bar_qfull + s, 2 * C::kQBytes);
        for (int c = 0; c < D / 64; ++c) {
          tma_load_4d(&tm_q, bar_qfull + s, qdst + c * (kTileM * 128), c * 64, qt * kTileM, h, b);
          tma_load_4d(&tm_do, bar_qfull + s, qdst + C::kQBytes + c * (kTileM * 128), c * 64,
                      qt * kTileM, h, b);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0 && any) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T, dO V^T
      constexpr uint32_t idesc_t = idesc_bf16(D, 64, 1, 1);    // dO^T A, Q^T dZ: both MN-major
      const uint32_t k_addr = smem_u32(smem + C::kOffK);
      const uint32_t v_addr = smem_u32(smem + C::kOffV);
      const uint32_t q0_addr = smem_u32(smem + C::kOffQ);
      const uint32_t a_addr = smem_u32(smem + C::kOffA);
      const uint32_t z_addr = smem_u32(smem + C::kOffZ);
      mbar_wait(bar_kv, 0);
      auto issue_kv = [&](int i) {
        const int s = i % ST;
        const uint32_t qa = q0_addr + s * 2 * C::kQBytes, da = qa + C::kQBytes;
        mbar_wait(bar_afull, i & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kTileM / 16; ++k)  // dV^T += dO^T A  (K = query rows)
          umma_ss(tbase + C::kColV, sdesc_sw128(da + k * 2048, kTileM * 128, 1024),
                  sdesc_sw128(a_addr + k * 2048, 16, 1024), idesc_t, (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(bar_aempty);
        mbar_wait(bar_zfull, i & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kTileM / 16; ++k)  // dK^T += Q^T dZ
          umma_ss(tbase + C::kColK, sdesc_sw128(qa + k * 2048, kTileM * 128, 1024),
                  sdesc_sw128(z_addr + k * 2048, 16, 1024), idesc_t, (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(bar_zempty);
        umma_commit(bar_qempty + s);
      };
      int j = 0;
      for (int qt = qt_first; qt < g.n_qt; qt = next_live_qt(fkb, g.nb, g.n_qt, kb, qt + 1), ++j) {
        const int s = j % ST;
        const uint32_t qa = q0_addr + s * 2 * C::kQBytes, da = qa + C::kQBytes;
        mbar_wait(bar_qfull + s, (j / ST) & 1);
        if (j >= 2) mbar_wait(bar_sempty + (j & 1), ((j >> 1) + 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
          const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
          umma_ss(tbase + C::kColS + (j & 1) * 64, sdesc_sw128(qa + off, 16, 1024),
                  sdesc_sw128(k_addr + offk, 16, 1024), idesc_s, k > 0);
        }
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
          const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
          umma_ss(tbase + C::kColW + (j & 1) * 64, sdesc_sw128(da + off, 16, 1024),
                  sdesc_sw128(v_addr + offk, 16, 1024), idesc_s, k > 0);
        }
        umma_commit(bar_sfull + (j & 1));
        if (j >= 1) issue_kv(j - 1);
      }
      issue_kv(j - 1);
      umma_commit(bar_done);
    }
  } else {
    const int quarter = warp & 3, gi = warp >> 2;
    const int r = quarter * 32 + lane;
    const int c0 = gi * kBwdCG;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const float* Mbase = args.M + unit * g.n_tiles * kBlock + (r & 63);
    const float* Nbase = args.N + unit * g.n_tiles * kBlock + (r & 63);
    const uint32_t a_row = smem_u32(smem + C::kOffA) + r * 128;
    const uint32_t z_row = smem_u32(smem + C::kOffZ) + r * 128;
    int j = 0;
    for (int qt = qt_first; qt < g.n_qt; qt = next_live_qt(fkb, g.nb, g.n_qt, kb, qt + 1), ++j) {
      const int par = j & 1;
      const int my_qb = 2 * qt + (r >> 6);
      const int row = qt * kTileM + r;
      const bool live = row < g.L && my_qb >= kb && fkb[my_qb] <= kb;
      const int lim = (kb == my_qb) ? (r & 63) : kBlock;
      const int64_t t = tile_index(my_qb, kb) * kBlock;
      float Ma = 0.0f, Nb = 0.0f, off = 0.0f;
      if (live) {
        Ma = Mbase[t];
        Nb = Nbase[t];
        off = args.row_offset ? args.row_offset[unit * g.L + row] : 0.0f;
      }
      mbar_wait(bar_sfull + par, (j >> 1) & 1);
      tc_fence_after();
      RowTile rt;
      tmem_ld16(tbase + lane_base + C::kColS + par * 64 + c0, rt.z);
      tmem_ld16(tbase + lane_base + C::kColW + par * 64 + c0, rt.w);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar_sempty + par);

      const bool diag = kb == my_qb;  // warp-uniform
      float part = 1.0f, right, left, tot;
      if (live)
        part = diag ? bwd_pass1<true>(rt, g.scale_log2, c0, lim)
                    : bwd_pass1<false>(rt, g.scale_log2, c0, lim);
      xch1[(par * kBwdGroups + gi) * 128 + r] = part;
      named_bar_sync(1, kBwdStick);
      right = exchange_right_prod(xch1, par, gi, r);
      uint32_t pa[kBwdCG / 2], pz[kBwdCG / 2];
      if (live) {
        part = bwd_pass2(rt, ex2(Ma) * right, off, pa);
      } else {
        part = 0.0f;
#pragma unroll
        for (int c = 0; c < kBwdCG / 2; ++c) pa[c] = 0u;
      }
      if (j >= 1) mbar_wait(bar_aempty, (j - 1) & 1);
      store_cols_sw128(a_row, r, gi, pa);
      fence_proxy_async_smem();
      mbar_arrive(bar_afull);
      xch2[(par * kBwdGroups + gi) * 128 + r] = part;
      named_bar_sync(1, kBwdStick);
      exchange_sums(xch2, par, gi, r, right, left, tot);
      if (live) {
        bwd_pass3(rt, left + Nb, pz);
      } else {
#pragma unroll
        for (int c = 0; c < kBwdCG / 2; ++c) pz[c] = 0u;
      }
      if (j >= 1) mbar_wait(bar_zempty, (j - 1) & 1);
      store_cols_sw128(z_row, r, gi, pz);
      fence_proxy_async_smem();
      mbar_arrive(bar_zfull);
    }

    // epilogue: TMEM holds dV^T / dK^T (lanes = head-dim index, columns = keys);
    // column group gi owns keys [16*gi, 16*gi+16).
    // M = 128: lane r <-> d = r.  M = 64: rows 16w+i live in lanes 32w+i, i < 16.
    const int dlane = (D == 128) ? r : (lane < 16 ? (quarter * 16 + lane) : -1);
    float vv[kBwdCG], kk[kBwdCG];
    if (any) {
      mbar_wait(bar_done, 0);
      tc_fence_after();
      tmem_ld16(tbase + lane_base + C::kColV + c0, vv);
      tmem_ld16(tbase + lane_base + C::kColK + c0, kk);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int c = 0; c < kBwdCG; ++c) vv[c] = kk[c] = 0.0f;
    }
    const float scale = g.scale_log2 * kLn2;
    const int64_t base = (int64_t)b * g.sb + (int64_t)h * g.sh;
    if (dlane >= 0) {
#pragma unroll
      for (int c = 0; c < kBwdCG; ++c) {
        const int key = kb * kBlock + c0 + c;
        if (key < g.L) {
          const int64_t o = base + (int64_t)key * g.sl + dlane;
          args.dv[o] = __float2bfloat16_rn(vv[c]);
          args.dk[o] = __float2bfloat16_rn(kk[c] * scale);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProdWarp) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D>
static int launch_bwd(const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk,
                      const CUtensorMap& tv, const BwdArgs& a, int phases, cudaStream_t stream) {
  if (phases & 1) {
    using C = BwdQCfg<D>;
    auto kern = sb_bwd_q_kernel<D>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return (int)e;
    kern<<<(unsigned)(a.g.n_qt * a.g.B * a.g.H), kBwdThreads, C::kSmem, stream>>>(tq, tdo, tk,
                                                                                   tv, a);
    if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  }
  if (phases & 2) {
    using C = BwdKVCfg<D>;
    auto kern = sb_bwd_kv_kernel<D>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return (int)e;
    kern<<<(unsigned)(a.g.nb * a.g.B * a.g.H), kBwdThreads, C::kSmem, stream>>>(tq, tdo, tk, tv,
                                                                                 a);
    if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  }
  return 0;
}

int bwd_dispatch(int D, const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk,
                 const CUtensorMap& tv, const BwdArgs& a, int phases, cudaStream_t stream) {
  if (D == 128) return launch_bwd<128>(tq, tdo, tk, tv, a, phases, stream);
  if (D == 64) return launch_bwd<64>(tq, tdo, tk, tv, a, phases, stream);
  return -1;
}

}  // namespace sb
