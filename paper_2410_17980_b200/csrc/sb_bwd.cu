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
// Both phases use the ping-pong layout of sb_fwd_pp.cu: two stick warpgroups
// per CTA (thread r <-> TMEM lane r <-> query row, all 64 key columns of a tile
// in registers), each with its own MMA-issuer thread and TMEM/smem buffers.
//   phase 1: WG w owns query tile 2p+w; both share one K/V stream.
//   phase 2: WG w owns key block 2p+w; both share one Q/dO stream.
// Tile math is the product form (sb_common.cuh): A_c = sigma_c * e^M *
// prod_{c'>c} r_c', sigma = t/(1+t), r = 1/(1+t): one ex2 + one rcp per element.
// Warps: 0-3 WG0, 4-7 WG1, 8 TMA producer (+TMEM allocator), 9/10 MMA for WG0/WG1,
// 11 idle; warpgroup 2 hands its registers to the stick warpgroups (setmaxnreg).
#include "sb_args.cuh"

namespace sb {

constexpr int kBwdThreads = 12 * 32;  // WG0, WG1 stick; WG2 = producer, MMA0, MMA1, idle
// setmaxnreg only redistributes the CTA's launch allocation (384 threads x 168
// registers): 128 x 56 + 256 x 224 == 384 x 168, otherwise .inc blocks forever.
constexpr int kRegsLaunch = 168, kRegsLow = 56, kRegsHigh = 224;
static_assert(128 * kRegsLow + 256 * kRegsHigh <= kBwdThreads * kRegsLaunch, "register budget");

// Right-to-left recompute of one row of a tile: on entry s[] = raw q.k dot
// products, on exit s[c] = A_c and sg[c] = sigma_c (both 0 where masked).
// E = e^M (the M snapshot in linear space).
template <bool kDiag>
__device__ __forceinline__ void recompute_row(float* s, float* sg, float scale_log2, float E,
                                              int lim) {
  float Ql = E;
#pragma unroll
  for (int c = kBlock - 1; c >= 0; --c) {
    const float Z = fminf(s[c] * scale_log2, 126.0f);  // t finite: sigma = t*r <= 1
    const float t = ex2(Z);
    float r = rcp(1.0f + t), sgm = t * r;
    if (kDiag && c >= lim) { r = 1.0f; sgm = 0.0f; }
    s[c] = sgm * Ql;
    sg[c] = sgm;
    Ql *= r;
  }
}

// dAt = A * (dW - off) with dW streamed from TMEM in 16-column chunks (warp-collective).
__device__ __forceinline__ void load_dat(float* s, uint32_t taddr, float off) {
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    float w[16];
    tmem_ld16(taddr + ch * 16, w);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 16; ++c) s[ch * 16 + c] *= (w[c] - off);
  }
}

// dZ = dAt - sigma*(prefix(dAt) + b), packed to bf16; returns rowsum(dAt).
__device__ __forceinline__ float dz_row(const float* dat, const float* sg, float b, uint32_t* pk) {
  float pfx = 0.0f;
#pragma unroll
  for (int c = 0; c < kBlock; c += 2) {
    pfx += dat[c];
    const float z0 = dat[c] - sg[c] * (pfx + b);
    pfx += dat[c + 1];
    const float z1 = dat[c + 1] - sg[c + 1] * (pfx + b);
    pk[c >> 1] = pack_bf16(z0, z1);
  }
  return pfx;
}

__device__ __forceinline__ void store_row_sw128(uint32_t row_addr, int r, const uint32_t* pk) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    st_shared_v4(row_addr + ((c ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                 pk[4 * c + 3]);
}

// ============================================================================
// Phase 1: dQ and N.  CTA = (b, h, query tiles 2p and 2p+1).
template <int D>
struct BwdQCfg {
  static constexpr int kStages = 2;
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kKVBytes = kBlock * D * 2;
  static constexpr int kZBytes = kTileM * kBlock * 2;
  static constexpr int kOffQ = 0;                       // Q[2]
  static constexpr int kOffDO = kOffQ + 2 * kQBytes;    // dO[2]
  static constexpr int kOffK = kOffDO + 2 * kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKVBytes;
  static constexpr int kOffZ = kOffV + kStages * kKVBytes;  // Z[2] (one per WG)
  static constexpr int kOffBar = kOffZ + 2 * kZBytes;
  static constexpr int kNumBars = 1 + 3 * kStages + 2 * 5;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static constexpr uint32_t kTmemCols = 512;  // per WG w at w*256: S +0, dW +64, dQ +128
};

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    sb_bwd_q_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const BwdArgs args) {
  using C = BwdQCfg<D>;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // heaviest pairs first (longest-processing-time order keeps the tail short)
  const int BH = g.B * g.H;
  const int n_pairs = (g.n_qt + 1) / 2;
  const int p = n_pairs - 1 - (int)(blockIdx.x / BH);
  const int bh = (int)(blockIdx.x % BH);
  const int b = bh / g.H, h = bh % g.H;
  const int64_t unit = (int64_t)b * g.H + h;
  const bool has1 = 2 * p + 1 < g.n_qt;
  const int kbhi0 = min(4 * p + 1, g.nb - 1);
  const int kbhi1 = has1 ? min(4 * p + 3, g.nb - 1) : kbhi0;
  const int* fkb = args.first_kb + unit * g.nb;
  int kb_lo = kbhi1;
  for (int qb = 4 * p; qb <= kbhi1; ++qb) kb_lo = min(kb_lo, fkb[qb]);
  const int n_s = kbhi1 - kb_lo + 1;  // stream tiles, kb = kb_lo .. kbhi1

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_qdo = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_vfull = bar_kfull + ST;
  uint64_t* bar_kvempty = bar_vfull + ST;
  uint64_t* wgbars = bar_kvempty + ST;  // per wg: sfull, sempty, zfull, zempty, done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);

  if (threadIdx.x == 0) {
    mbar_init(bar_qdo, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_kfull + s, 1);
      mbar_init(bar_vfull + s, 1);
      mbar_init(bar_kvempty + s, has1 ? 2 : 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(wgbars + w * 5 + 0, 1);
      mbar_init(wgbars + w * 5 + 1, 128);
      mbar_init(wgbars + w * 5 + 2, 128);
      mbar_init(wgbars + w * 5 + 3, 1);
      mbar_init(wgbars + w * 5 + 4, 1);
    }
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp >= 8) {
    reg_dealloc<kRegsLow>();
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_do);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      const int nw = has1 ? 2 : 1;
      mbar_expect_tx(bar_qdo, nw * 2 * C::kQBytes);
      for (int w = 0; w < nw; ++w)
        for (int c = 0; c < D / 64; ++c) {
          const int row0 = (2 * p + w) * kTileM;
          tma_load_4d(&tm_q, bar_qdo, smem + C::kOffQ + w * C::kQBytes + c * (kTileM * 128),
                      c * 64, row0, h, b);
          tma_load_4d(&tm_do, bar_qdo, smem + C::kOffDO + w * C::kQBytes + c * (kTileM * 128),
                      c * 64, row0, h, b);
        }
      for (int j = 0; j < n_s; ++j) {
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
  } else if (warp == 9 || warp == 10) {
    const int w = warp - 9;
    if (lane == 0 && (w == 0 || has1)) {
      uint64_t* sfull = wgbars + w * 5;
      uint64_t* sempty = sfull + 1;
      uint64_t* zfull = sfull + 2;
      uint64_t* zempty = sfull + 3;
      uint64_t* done = sfull + 4;
      constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T, dO V^T
      constexpr uint32_t idesc_q = idesc_bf16(128, D, 0, 1);   // dZ K: K is MN-major
      const uint32_t q_addr = smem_u32(smem + C::kOffQ + w * C::kQBytes);
      const uint32_t do_addr = smem_u32(smem + C::kOffDO + w * C::kQBytes);
      const uint32_t k_addr = smem_u32(smem + C::kOffK);
      const uint32_t v_addr = smem_u32(smem + C::kOffV);
      const uint32_t z_addr = smem_u32(smem + C::kOffZ + w * C::kZBytes);
      const uint32_t tS = tbase + w * 256, tW = tS + 64, tQ = tS + 128;
      const int n_w = (w ? kbhi1 : kbhi0) - kb_lo + 1;
      mbar_wait(bar_qdo, 0);
      auto issue_dq = [&](int i) {  // inputs landed
        const int s = i % ST;
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kBlock / 16; ++k)
          umma_ss(tQ, sdesc_sw128(z_addr + k * 32, 16, 1024),
                  sdesc_sw128(k_addr + s * C::kKVBytes + k * 2048, kBlock * 128, 1024), idesc_q,
                  (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(zempty);
        umma_commit(bar_kvempty + s);
      };
      // two in-order queues (S and dW, then dQ), issued as their inputs land
      int is = 0, iq = 0;
      while (iq < n_w) {
        const int progress = is + iq;
        if (is < n_w) {
          const int s = is % ST;
          if (mbar_test(bar_kfull + s, (is / ST) & 1) && mbar_test(bar_vfull + s, (is / ST) & 1) &&
              (is < 1 || mbar_test(sempty, (is - 1) & 1))) {
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
              const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
              umma_ss(tS, sdesc_sw128(q_addr + off, 16, 1024),
                      sdesc_sw128(k_addr + s * C::kKVBytes + offk, 16, 1024), idesc_s, k > 0);
            }
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
              const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
              umma_ss(tW, sdesc_sw128(do_addr + off, 16, 1024),
                      sdesc_sw128(v_addr + s * C::kKVBytes + offk, 16, 1024), idesc_s, k > 0);
            }
            umma_commit(sfull);
            ++is;
          }
        }
        if (iq < is && mbar_test(zfull, iq & 1)) {
          issue_dq(iq);
          ++iq;
        }
        if (is + iq == progress) __nanosleep(32);  // nothing ready: yield the SMSP
      }
      umma_commit(done);
      for (int j = n_w; j < n_s; ++j) {  // stream tiles right of this WG's diagonal
        mbar_wait(bar_vfull + j % ST, (j / ST) & 1);
        mbar_arrive(bar_kvempty + j % ST);
      }
    }
  }
  } else {
    reg_alloc<kRegsHigh>();
    const int w = warp >> 2;
    if (w == 0 || has1) {
      uint64_t* sfull = wgbars + w * 5;
      uint64_t* sempty = sfull + 1;
      uint64_t* zfull = sfull + 2;
      uint64_t* zempty = sfull + 3;
      uint64_t* done = sfull + 4;
      const int quarter = warp & 3;
      const int r = quarter * 32 + lane;
      const int qt = 2 * p + w;
      const int my_qb = 2 * qt + (r >> 6);
      const int row = qt * kTileM + r;
      const bool row_valid = row < g.L;
      const bool half_exists = my_qb < g.nb;
      const int my_first = half_exists ? fkb[my_qb] : g.nb;
      const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
      const uint32_t tS = tbase + w * 256 + lane_base, tW = tS + 64, tQ = tS + 128;
      const float off = (args.row_offset && row_valid) ? args.row_offset[unit * g.L + row] : 0.0f;
      const float* Mrow = args.M + unit * g.n_tiles * kBlock + (r & 63);
      float* Nrow = args.N + unit * g.n_tiles * kBlock + (r & 63);
      const uint32_t z_row = smem_u32(smem + C::kOffZ + w * C::kZBytes) + r * 128;
      const int n_w = (w ? kbhi1 : kbhi0) - kb_lo + 1;
      float bsum = 0.0f;  // running b (blocked.py:342, :354)
      for (int j = 0; j < n_w; ++j) {
        const int kb = kb_lo + j;
        const bool live = row_valid && kb >= my_first && kb <= my_qb;
        const int64_t t = tile_index(live ? my_qb : 0, live ? kb : 0) * kBlock;
        const float Ma = Mrow[t];  // issued before the S wait to hide its latency
        mbar_wait(sfull, j & 1);
        tc_fence_after();
        float s[64], sg[64];
        tmem_ld32(tS, s);
        tmem_ld32(tS + 32, s + 32);
        tmem_wait_ld();
        const bool diag = kb == my_qb;  // warp-uniform
        if (live) {
          if (diag) recompute_row<true>(s, sg, g.scale_log2, ex2(Ma), r & 63);
          else recompute_row<false>(s, sg, g.scale_log2, ex2(Ma), kBlock);
        } else {
#pragma unroll
          for (int c = 0; c < kBlock; ++c) s[c] = sg[c] = 0.0f;
        }
        load_dat(s, tW, off);
        tc_fence_before();
        mbar_arrive(sempty);
        uint32_t pk[32];
        if (live) {
          Nrow[t] = bsum;  // b in effect for this tile (blocked.py:353)
          bsum += dz_row(s, sg, bsum, pk);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = 0u;
        }
        if (j >= 1) mbar_wait(zempty, (j - 1) & 1);
        store_row_sw128(z_row, r, pk);
        fence_proxy_async_smem();
        mbar_arrive(zfull);
      }
      mbar_wait(done, 0);
      tc_fence_after();
      const float scale = g.scale_log2 * kLn2;
      __nv_bfloat16* dqrow = args.dq + (int64_t)b * g.sb + (int64_t)h * g.sh + (int64_t)row * g.sl;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float v[32];
        tmem_ld32(tQ + c * 32, v);
        tmem_wait_ld();
        if (row_valid) {
          uint4* dst = reinterpret_cast<uint4*>(dqrow + c * 32);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            dst[q4] = make_uint4(pack_bf16(v[8 * q4] * scale, v[8 * q4 + 1] * scale),
                                 pack_bf16(v[8 * q4 + 2] * scale, v[8 * q4 + 3] * scale),
                                 pack_bf16(v[8 * q4 + 4] * scale, v[8 * q4 + 5] * scale),
                                 pack_bf16(v[8 * q4 + 6] * scale, v[8 * q4 + 7] * scale));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc<C::kTmemCols>(tbase);
}

// ============================================================================
// Phase 2: dK and dV.  CTA = (b, h, key blocks 2p and 2p+1); query tiles stream.
template <int D>
struct BwdKVCfg {
  static constexpr int kStages = D == 128 ? 2 : 3;
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kKVBytes = kBlock * D * 2;
  static constexpr int kPBytes = kTileM * kBlock * 2;
  static constexpr int kOffK = 0;                               // K[2]
  static constexpr int kOffV = kOffK + 2 * kKVBytes;            // V[2]
  static constexpr int kOffQ = kOffV + 2 * kKVBytes;            // stage s: Q, dO
  static constexpr int kOffAZ = kOffQ + kStages * 2 * kQBytes;  // A then dZ, one per WG
  static constexpr int kOffBar = kOffAZ + 2 * kPBytes;
  static constexpr int kNumBars = 1 + 2 * kStages + 2 * 7;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static constexpr uint32_t kTmemCols = 512;  // per WG w at w*256: S +0, dW +64, dV^T +128, dK^T +192
};

// a tile (qb, kb) is live when the forward visited it: first_kb[qb] <= kb <= qb
// (blocked.py:372-373)
__device__ __forceinline__ bool tile_live(const int* fkb, int nb, int qb, int kb) {
  return qb < nb && qb >= kb && fkb[qb] <= kb;
}

// first query tile >= qt holding a live tile for key block kb0 or kb0+1
__device__ __forceinline__ int next_live_qt(const int* fkb, int nb, int n_qt, int kb0, int qt) {
  for (; qt < n_qt; ++qt)
    if (tile_live(fkb, nb, 2 * qt, kb0) || tile_live(fkb, nb, 2 * qt + 1, kb0) ||
        tile_live(fkb, nb, 2 * qt, kb0 + 1) || tile_live(fkb, nb, 2 * qt + 1, kb0 + 1))
      return qt;
  return n_qt;
}

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    sb_bwd_kv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                     const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     const BwdArgs args) {
  using C = BwdKVCfg<D>;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // small key blocks first: they own the longest columns (LPT order)
  const int BH = g.B * g.H;
  const int p = (int)(blockIdx.x / BH);
  const int bh = (int)(blockIdx.x % BH);
  const int b = bh / g.H, h = bh % g.H;
  const int64_t unit = (int64_t)b * g.H + h;
  const int kb0 = 2 * p;
  const bool has1 = kb0 + 1 < g.nb;
  const int* fkb = args.first_kb + unit * g.nb;
  const int qt_first = next_live_qt(fkb, g.nb, g.n_qt, kb0, p);

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_kv = bars;
  uint64_t* bar_qfull = bars + 1;
  uint64_t* bar_qempty = bar_qfull + ST;
  uint64_t* wgbars = bar_qempty + ST;  // per wg: sfull, sempty, afull, aused, zfull, zused, done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_qfull + s, 1);
      mbar_init(bar_qempty + s, has1 ? 2 : 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(wgbars + w * 7 + 0, 1);    // sfull
      mbar_init(wgbars + w * 7 + 1, 128);  // sempty
      mbar_init(wgbars + w * 7 + 2, 128);  // afull
      mbar_init(wgbars + w * 7 + 3, 1);    // aused (dV^T MMA read A)
      mbar_init(wgbars + w * 7 + 4, 128);  // zfull
      mbar_init(wgbars + w * 7 + 5, 1);    // zused (dK^T MMA read dZ)
      mbar_init(wgbars + w * 7 + 6, 1);    // done
    }
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const bool any = qt_first < g.n_qt;

  if (warp >= 8) {
    reg_dealloc<kRegsLow>();
  if (warp == 8) {
    if (lane == 0 && any) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_do);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      const int nw = has1 ? 2 : 1;
      mbar_expect_tx(bar_kv, nw * 2 * C::kKVBytes);
      for (int w = 0; w < nw; ++w)
        for (int c = 0; c < D / 64; ++c) {
          const int kr = (kb0 + w) * kBlock;
          tma_load_4d(&tm_k, bar_kv, smem + C::kOffK + w * C::kKVBytes + c * (kBlock * 128),
                      c * 64, kr, h, b);
          tma_load_4d(&tm_v, bar_kv, smem + C::kOffV + w * C::kKVBytes + c * (kBlock * 128),
                      c * 64, kr, h, b);
        }
      int j = 0;
      for (int qt = qt_first; qt < g.n_qt; qt = next_live_qt(fkb, g.nb, g.n_qt, kb0, qt + 1), ++j) {
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
  } else if (warp == 9 || warp == 10) {
    const int w = warp - 9;
    if (lane == 0 && any && (w == 0 || has1)) {
      uint64_t* sfull = wgbars + w * 7;
      uint64_t *sempty = sfull + 1, *afull = sfull + 2, *aused = sfull + 3, *zfull = sfull + 4,
               *zused = sfull + 5, *done = sfull + 6;
      constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T, dO V^T
      constexpr uint32_t idesc_t = idesc_bf16(D, 64, 1, 1);    // dO^T A, Q^T dZ: both MN-major
      const uint32_t k_addr = smem_u32(smem + C::kOffK + w * C::kKVBytes);
      const uint32_t v_addr = smem_u32(smem + C::kOffV + w * C::kKVBytes);
      const uint32_t q0_addr = smem_u32(smem + C::kOffQ);
      const uint32_t az_addr = smem_u32(smem + C::kOffAZ + w * C::kPBytes);
      const uint32_t tS = tbase + w * 256, tW = tS + 64, tV = tS + 128, tK = tS + 192;
      mbar_wait(bar_kv, 0);
      int n = 0;
      for (int qt = qt_first; qt < g.n_qt; qt = next_live_qt(fkb, g.nb, g.n_qt, kb0, qt + 1)) ++n;
      // three in-order queues (S and dW; dV^T += dO^T A; dK^T += Q^T dZ), issued
      // as their inputs land
      int is = 0, iv = 0, ik = 0;
      while (ik < n) {
        const int progress = is + iv + ik;
        if (is < n) {
          const int s = is % ST;
          if (mbar_test(bar_qfull + s, (is / ST) & 1) && (is < 1 || mbar_test(sempty, (is - 1) & 1))) {
            const uint32_t qa = q0_addr + s * 2 * C::kQBytes, da = qa + C::kQBytes;
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
              const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
              umma_ss(tS, sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(k_addr + offk, 16, 1024),
                      idesc_s, k > 0);
            }
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
              const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
              umma_ss(tW, sdesc_sw128(da + off, 16, 1024), sdesc_sw128(v_addr + offk, 16, 1024),
                      idesc_s, k > 0);
            }
            umma_commit(sfull);
            ++is;
          }
        }
        if (iv < is && mbar_test(afull, iv & 1)) {
          const uint32_t da = q0_addr + (iv % ST) * 2 * C::kQBytes + C::kQBytes;
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < kTileM / 16; ++k)  // dV^T += dO^T A  (K = query rows)
            umma_ss(tV, sdesc_sw128(da + k * 2048, kTileM * 128, 1024),
                    sdesc_sw128(az_addr + k * 2048, 16, 1024), idesc_t,
                    (iv > 0 || k > 0) ? 1u : 0u);
          umma_commit(aused);
          ++iv;
        }
        if (ik < iv && mbar_test(zfull, ik & 1)) {
          const int s = ik % ST;
          const uint32_t qa = q0_addr + s * 2 * C::kQBytes;
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < kTileM / 16; ++k)  // dK^T += Q^T dZ
            umma_ss(tK, sdesc_sw128(qa + k * 2048, kTileM * 128, 1024),
                    sdesc_sw128(az_addr + k * 2048, 16, 1024), idesc_t,
                    (ik > 0 || k > 0) ? 1u : 0u);
          umma_commit(zused);
          umma_commit(bar_qempty + s);
          ++ik;
        }
        if (is + iv + ik == progress) __nanosleep(32);  // nothing ready: yield the SMSP
      }
      umma_commit(done);
    }
  }
  } else {
    reg_alloc<kRegsHigh>();
    const int w = warp >> 2;
    if (w == 0 || has1) {
      uint64_t* sfull = wgbars + w * 7;
      uint64_t *sempty = sfull + 1, *afull = sfull + 2, *aused = sfull + 3, *zfull = sfull + 4,
               *zused = sfull + 5, *done = sfull + 6;
      const int quarter = warp & 3;
      const int r = quarter * 32 + lane;
      const int kb = kb0 + w;
      const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
      const uint32_t tS = tbase + w * 256 + lane_base, tW = tS + 64, tV = tS + 128, tK = tS + 192;
      const float* Mbase = args.M + unit * g.n_tiles * kBlock + (r & 63);
      const float* Nbase = args.N + unit * g.n_tiles * kBlock + (r & 63);
      const uint32_t az_row = smem_u32(smem + C::kOffAZ + w * C::kPBytes) + r * 128;
      int j = 0;
      for (int qt = qt_first; qt < g.n_qt; qt = next_live_qt(fkb, g.nb, g.n_qt, kb0, qt + 1), ++j) {
        const int my_qb = 2 * qt + (r >> 6);
        const int row = qt * kTileM + r;
        const bool live = row < g.L && tile_live(fkb, g.nb, my_qb, kb);
        const int64_t t = live ? tile_index(my_qb, kb) * kBlock : 0;
        const float Ma = Mbase[t], Nb = Nbase[t];  // issued before the S wait
        const float off = (live && args.row_offset) ? args.row_offset[unit * g.L + row] : 0.0f;
        mbar_wait(sfull, j & 1);
        tc_fence_after();
        float s[64], sg[64];
        tmem_ld32(tS, s);
        tmem_ld32(tS + 32, s + 32);
        tmem_wait_ld();
        const bool diag = kb == my_qb;  // warp-uniform
        if (live) {
          if (diag) recompute_row<true>(s, sg, g.scale_log2, ex2(Ma), r & 63);
          else recompute_row<false>(s, sg, g.scale_log2, ex2(Ma), kBlock);
        } else {
#pragma unroll
          for (int c = 0; c < kBlock; ++c) s[c] = sg[c] = 0.0f;
        }
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) pk[c] = pack_bf16(s[2 * c], s[2 * c + 1]);
        if (j >= 1) mbar_wait(zused, (j - 1) & 1);  // dK^T of the previous tile read the buffer
        store_row_sw128(az_row, r, pk);
        fence_proxy_async_smem();
        mbar_arrive(afull);
        load_dat(s, tW, off);  // warp-collective
        tc_fence_before();
        mbar_arrive(sempty);
        if (live) {
          dz_row(s, sg, Nb, pk);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = 0u;
        }
        mbar_wait(aused, j & 1);  // dV^T of this tile read A
        store_row_sw128(az_row, r, pk);
        fence_proxy_async_smem();
        mbar_arrive(zfull);
      }

      // epilogue: dV^T / dK^T in TMEM (lanes = head-dim index, columns = keys of kb).
      // M = 128: lane r <-> d = r.  M = 64: rows 16q+i live in lanes 32q+i, i < 16.
      const int dlane = (D == 128) ? r : (lane < 16 ? (quarter * 16 + lane) : -1);
      if (any) {
        mbar_wait(done, 0);
        tc_fence_after();
      }
      const float scale = g.scale_log2 * kLn2;
      const int64_t base = (int64_t)b * g.sb + (int64_t)h * g.sh;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float vv[32], kk[32];
        if (any) {
          tmem_ld32(tV + half * 32, vv);
          tmem_ld32(tK + half * 32, kk);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) vv[c] = kk[c] = 0.0f;
        }
        if (dlane >= 0) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int key = kb * kBlock + half * 32 + c;
            if (key < g.L) {
              const int64_t o = base + (int64_t)key * g.sl + dlane;
              args.dv[o] = __float2bfloat16_rn(vv[c]);
              args.dk[o] = __float2bfloat16_rn(kk[c] * scale);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D>
static int launch_bwd(const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk,
                      const CUtensorMap& tv, const BwdArgs& a, int phases, cudaStream_t stream) {
  const unsigned BH = (unsigned)(a.g.B * a.g.H);
  if (phases & 1) {
    using C = BwdQCfg<D>;
    auto kern = sb_bwd_q_kernel<D>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return (int)e;
    kern<<<(unsigned)((a.g.n_qt + 1) / 2) * BH, kBwdThreads, C::kSmem, stream>>>(tq, tdo, tk, tv,
                                                                                  a);
    if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  }
  if (phases & 2) {
    using C = BwdKVCfg<D>;
    auto kern = sb_bwd_kv_kernel<D>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return (int)e;
    kern<<<(unsigned)((a.g.nb + 1) / 2) * BH, kBwdThreads, C::kSmem, stream>>>(tq, tdo, tk, tv,
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
