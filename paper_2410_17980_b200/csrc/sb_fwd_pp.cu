// Stick-breaking attention forward, ping-pong variant (skip off), sm_100a.
//
// Same algorithm as sb_fwd.cu (reference blocked.py:129-206, two_phase=True),
// organised for throughput: one CTA owns TWO 128-row query tiles of the same
// (b, h) (tiles 2p and 2p+1, i.e. four reference query blocks) and streams the
// shared K/V blocks right to left once. Each query tile has its own stick
// warpgroup (WG0 / WG1, thread r <-> TMEM lane r <-> query row), its own
// MMA-issuer thread and its own S/P buffers, so the two warpgroups interleave
// on every SMSP without any cross-warpgroup synchronisation; each thread scans
// all 64 key columns of its row in registers.
//
// Per element (product form, sb_common.cuh): t = 2^Z, r = 1/(1+t), sigma = t*r,
// A = sigma * (e^a * prod of r to the right), i.e. one ex2 + one rcp.  The
// row total of lt for `a` is one lg2 of the tile's product of r (exact
// softplus sum if that product underflows).
//
// Warps: 0-3 WG0, 4-7 WG1, 8 TMA producer (+TMEM allocator), 9 MMA for WG0,
// 10 MMA for WG1.
#include "sb_args.cuh"

namespace sb {

template <int D>
struct FwdPPCfg {
  static constexpr int kStages = D == 128 ? 3 : 4;
  static constexpr int kThreads = 11 * 32;
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kKVBytes = kBlock * D * 2;
  static constexpr int kPBytes = kTileM * kBlock * 2;
  static constexpr int kOffQ = 0;                                // Q[2]
  static constexpr int kOffK = kOffQ + 2 * kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKVBytes;
  static constexpr int kOffP = kOffV + kStages * kKVBytes;       // P[wg][buf]
  static constexpr int kOffBar = kOffP + 4 * kPBytes;
  static constexpr int kNumBars = 1 + 3 * kStages + 2 * 8 + 2;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static constexpr uint32_t kTmemCols = 512;  // S[wg][2] at wg*128 + b*64, O[wg] at 256 + wg*128
};

template <int D>
__global__ void __launch_bounds__(FwdPPCfg<D>::kThreads, 1)
    sb_fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const FwdArgs args) {
  using C = FwdPPCfg<D>;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // pair p covers query tiles 2p (WG0) and 2p+1 (WG1); heaviest pairs first
  // (longest-processing-time order keeps the tail short)
  const int BH = g.B * g.H;
  int item, bh;
  grouped_order((int)blockIdx.x, (g.n_qt + 1) / 2, BH, item, bh);
  const int b = bh / g.H, h = bh % g.H;
  const Unit u = make_unit(g, b, h);
  const int n_pairs = (u.n_qt + 1) / 2;
  if (item >= n_pairs) return;  // shorter sequence of a varlen batch: no work
  const int p = n_pairs - 1 - item;
  const bool has1 = 2 * p + 1 < u.n_qt;
  const int kbhi0 = min(4 * p + 1, u.nb - 1);
  const int kbhi1 = has1 ? min(4 * p + 3, u.nb - 1) : kbhi0;
  const int n_s = kbhi1 + 1;  // stream tiles, kb = kbhi1 .. 0

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_vfull = bar_kfull + ST;
  uint64_t* bar_kvempty = bar_vfull + ST;
  uint64_t* wgbars = bar_kvempty + ST;  // per wg: sfull[2], sempty[2], pfull[2], pempty[2]
  uint64_t* bar_ofull = wgbars + 16;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_kfull + s, 1);
      mbar_init(bar_vfull + s, 1);
      mbar_init(bar_kvempty + s, has1 ? 2 : 1);
    }
    for (int w = 0; w < 2; ++w)
      for (int s = 0; s < 2; ++s) {
        mbar_init(wgbars + w * 8 + 0 + s, 1);    // sfull
        mbar_init(wgbars + w * 8 + 2 + s, 128);  // sempty
        mbar_init(wgbars + w * 8 + 4 + s, 128);  // pfull
        mbar_init(wgbars + w * 8 + 6 + s, 1);    // pempty
      }
    mbar_init(bar_ofull, 1);
    mbar_init(bar_ofull + 1, 1);
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      mbar_expect_tx(bar_q, (has1 ? 2 : 1) * C::kQBytes);
      for (int w = 0; w < (has1 ? 2 : 1); ++w)
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_q, bar_q, smem + C::kOffQ + w * C::kQBytes + c * (kTileM * 128), c * 64,
                      u.trow0 + (2 * p + w) * kTileM, h, u.tb);
      for (int j = 0; j < n_s; ++j) {
        const int s = j % ST;
        if (j >= ST) mbar_wait(bar_kvempty + s, ((j / ST) - 1) & 1);
        const int kb = kbhi1 - j;
        mbar_expect_tx(bar_kfull + s, C::kKVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_k, bar_kfull + s, smem + C::kOffK + s * C::kKVBytes + c * (kBlock * 128),
                      c * 64, u.trow0 + kb * kBlock, h, u.tb);
        mbar_expect_tx(bar_vfull + s, C::kKVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_v, bar_vfull + s, smem + C::kOffV + s * C::kKVBytes + c * (kBlock * 128),
                      c * 64, u.trow0 + kb * kBlock, h, u.tb);
      }
    }
  } else if (warp == 9 || warp == 10) {
    // ------------------------------------------------------------ MMA issuer of one WG
    // The whole warp runs the (uniform) control flow and computes descriptors in
    // uniform registers; one elected lane issues the MMAs and their commits.
    const int w = warp - 9;
    if (w == 0 || has1) {
      uint64_t* sfull = wgbars + w * 8;
      uint64_t* sempty = sfull + 2;
      uint64_t* pfull = sfull + 4;
      uint64_t* pempty = sfull + 6;
      constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T: both K-major
      constexpr uint32_t idesc_o = idesc_bf16(128, D, 0, 1);   // A V: V is MN-major
      const uint64_t dq = sdesc_sw128(smem_u32(smem + C::kOffQ + w * C::kQBytes), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(smem + C::kOffK), 16, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(smem + C::kOffV), kBlock * 128, 1024);
      const uint64_t dp = sdesc_sw128(smem_u32(smem + C::kOffP + w * 2 * C::kPBytes), 16, 1024);
      const uint32_t tS = tbase + w * 128, tO = tbase + 256 + w * 128;
      const int j0 = kbhi1 - (w ? kbhi1 : kbhi0);  // first stream tile of this WG
      const int n_w = n_s - j0;
      const bool leader = elect_one();
      mbar_wait(bar_q, 0);
      auto issue_pv = [&](int i) {  // local tile i == stream tile j0 + i
        const int s = (j0 + i) % ST;
        mbar_wait(pfull + (i & 1), (i >> 1) & 1);
        SB_TR(args, 2 + w, i, 9);
        mbar_wait(bar_vfull + s, ((j0 + i) / ST) & 1);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int k = 0; k < kBlock / 16; ++k)
            umma_ss(tO, desc_add(dp, (i & 1) * C::kPBytes + k * 32),
                    desc_add(dv, s * C::kKVBytes + k * 2048), idesc_o, (i > 0 || k > 0) ? 1u : 0u);
          umma_commit(pempty + (i & 1));
          umma_commit(bar_kvempty + s);
        }
        __syncwarp();
        SB_TR(args, 2 + w, i, 11);
      };
      for (int j = 0; j < j0; ++j) {  // stream tiles right of this WG's diagonal
        mbar_wait(bar_vfull + j % ST, (j / ST) & 1);
        if (leader) mbar_arrive(bar_kvempty + j % ST);
      }
      for (int i = 0; i < n_w; ++i) {
        const int j = j0 + i, s = j % ST;
        mbar_wait(bar_kfull + s, (j / ST) & 1);
        if (i >= 2) mbar_wait(sempty + (i & 1), ((i >> 1) + 1) & 1);
        SB_TR(args, 2 + w, i, 8);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
            umma_ss(tS + (i & 1) * 64, desc_add(dq, off), desc_add(dk, s * C::kKVBytes + offk),
                    idesc_s, k > 0);
          }
          umma_commit(sfull + (i & 1));
        }
        __syncwarp();
        SB_TR(args, 2 + w, i, 10);
        if (i >= 1) issue_pv(i - 1);
      }
      issue_pv(n_w - 1);
      if (leader) umma_commit(bar_ofull + w);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ stick warpgroups
    const int w = warp >> 2;
    if (w == 0 || has1) {
      uint64_t* sfull = wgbars + w * 8;
      uint64_t* sempty = sfull + 2;
      uint64_t* pfull = sfull + 4;
      uint64_t* pempty = sfull + 6;
      const int quarter = warp & 3;
      const int r = quarter * 32 + lane;
      const int qt = 2 * p + w;
      const int my_qb = 2 * qt + (r >> 6);
      const int row = qt * kTileM + r;
      const bool row_valid = row < u.L;
      const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
      const uint32_t tS = tbase + w * 128 + lane_base, tO = tbase + 256 + w * 128 + lane_base;
      float* Mrow = args.M + u.m_off + (r & 63);
      const uint32_t p_row = smem_u32(smem + C::kOffP + w * 2 * C::kPBytes) + r * 128;
      const int kbhi = w ? kbhi1 : kbhi0;
      const int n_w = kbhi + 1;
      const float sl2 = g.scale_log2;
      float a2 = 0.0f;  // running log2 remaining mass
      const bool tr = quarter == 0 && lane == 0;
      if (tr) SB_TR(args, w, 0, 14);
      for (int i = 0; i < n_w; ++i) {
        const int kb = kbhi - i;
        if (tr) SB_TR(args, w, i, 0);
        mbar_wait(sfull + (i & 1), (i >> 1) & 1);
        tc_fence_after();
        float s[64];
        tmem_ld32(tS + (i & 1) * 64, s);
        tmem_ld32(tS + (i & 1) * 64 + 32, s + 32);
        tmem_wait_ld();
        if (tr) SB_TR(args, w, i, 1);
        uint32_t pk[32];
        bool slow = false;
        const bool diag = kb == my_qb;
        const int lim = diag ? (r & 63) : kBlock;
        if (kb <= my_qb) {  // warp-uniform: a warp's rows share one 64-row half
          // batched reciprocal (sb_common.cuh): one rcp per 16 columns
          float Q = ex2(a2), Dhi = 1.0f, Dlo = 1.0f;
          slow = diag ? !batched_row<true>(s, pk, sl2, lim, Q, Dhi, Dlo)
                      : !batched_row<false>(s, pk, sl2, kBlock, Q, Dhi, Dlo);
          if (row_valid) Mrow[tile_index(my_qb, kb) * kBlock] = a2;
          if (!slow) a2 -= lg2(Dhi) + lg2(Dlo);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = 0u;
        }
        if (__any_sync(0xffffffffu, slow)) {
          // the tile consumed more than 2^-120 of some row's stick: exact sum of
          // lt for those rows (S is still in TMEM: s_empty not yet signalled)
          tmem_ld32(tS + (i & 1) * 64, s);
          tmem_ld32(tS + (i & 1) * 64 + 32, s + 32);
          tmem_wait_ld();
          if (slow) {
            // per-element product form for A, exact softplus sum for a
            float Ql = ex2(a2), lt = 0.0f;
#pragma unroll
            for (int c = kBlock - 1; c >= 0; c -= 2) {
              float A[2];
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int cc = c - u;
                const float Z = fminf(s[cc] * sl2, 126.0f);  // t finite: sigma = t*r <= 1
                const float t = ex2(Z);
                float rr = rcp(1.0f + t), sg = t * rr;
                const float sp = softplus2(s[cc] * sl2, t);
                if (cc >= lim) { rr = 1.0f; sg = 0.0f; }
                lt -= (cc < lim) ? sp : 0.0f;
                A[u] = sg * Ql;
                Ql *= rr;
              }
              pk[(c - 1) >> 1] = pack_bf16(A[1], A[0]);
            }
            a2 += lt;
          }
        }
        tc_fence_before();
        mbar_arrive(sempty + (i & 1));
        if (tr) SB_TR(args, w, i, 2);
        if (i >= 2) mbar_wait(pempty + (i & 1), ((i >> 1) + 1) & 1);
        if (tr) SB_TR(args, w, i, 3);
        const uint32_t pb = p_row + (i & 1) * C::kPBytes;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          st_shared_v4(pb + ((c ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                       pk[4 * c + 3]);
        fence_proxy_async_smem();
        mbar_arrive(pfull + (i & 1));
        if (tr) SB_TR(args, w, i, 4);
      }
      // epilogue
      mbar_wait(bar_ofull + w, 0);
      tc_fence_after();
      // O rows leave in 64-column halves through this warp's 4 KB slice of the
      // (now idle: ofull) P buffers as coalesced row segments
      const int row0 = qt * kTileM + quarter * 32;
      const int nvalid = max(0, min(32, u.L - row0));
      const uint32_t stage = smem_u32(smem + C::kOffP + w * 2 * C::kPBytes) + quarter * 4096;
#pragma unroll 1
      for (int c = 0; c < D / 64; ++c) {
        float ov[64];
        tmem_ld32(tO + c * 64, ov);
        tmem_ld32(tO + c * 64 + 32, ov + 32);
        tmem_wait_ld();
        warp_store_rows<8>(ov, 1.0f, stage, args.o + u.out_off + (int64_t)row0 * g.sl + c * 64,
                           g.sl, nvalid);
      }
      if (row_valid) args.log_rem[u.rem_off + row * u.rem_stride] = a2 * kLn2;
      if (my_qb < u.nb && (r & 63) == 0) {
        args.first_kb[u.fkb_off + my_qb] = 0;
        if (args.counters) atomicAdd(args.counters, (unsigned long long)(my_qb + 1));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D>
static int launch_fwd_pp(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const FwdArgs& a, cudaStream_t stream) {
  using C = FwdPPCfg<D>;
  auto kern = sb_fwd_pp_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  if (e != cudaSuccess) return (int)e;
  const unsigned grid = (unsigned)(((a.g.n_qt + 1) / 2) * a.g.B * a.g.H);
  kern<<<grid, C::kThreads, C::kSmem, stream>>>(tq, tk, tv, a);
  return (int)cudaGetLastError();
}

int fwd_pp_dispatch(int D, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                    const FwdArgs& a, cudaStream_t stream) {
  if (D == 128) return launch_fwd_pp<128>(tq, tk, tv, a, stream);
  if (D == 64) return launch_fwd_pp<64>(tq, tk, tv, a, stream);
  return -1;
}

}  // namespace sb
