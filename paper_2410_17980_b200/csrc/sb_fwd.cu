// Stick-breaking attention forward (K1 of SURVEY.md §2.2) for sm_100a.
//
// Restates blocked_forward (reference blocked.py:129-206, two_phase=True):
// per query block, key blocks right to left,
//     z = q k^T * scale,  lt = -softplus(z) (0 where masked),
//     A = exp(z + suffix_cumsum(lt) + a),  O += A V,  a += rowsum(lt)
// with the optional skip check `max_rows(a) < log(eps)` before every key
// block left of the diagonal (blocked.py:175-176), M snapshots (a in effect per
// tile, blocked.py:188-189) and first_kb (blocked.py:192, :202).
//
// One CTA = one (b, h, 128-row query tile) = two reference query blocks
// (64-row skip groups). Warp roles:
//   warps 0..4*NG-1  "stick" warps. Warp w owns TMEM lanes (= query rows)
//              32*(w%4)..+31 and key columns [CG*(w/4), CG*(w/4)+CG) of every
//              64-column S tile (CG = 64/NG). Each thread scans its CG columns
//              right to left in registers; the NG column groups of a row combine
//              their partial suffix sums of lt through shared memory (one named
//              barrier per tile), then write A (bf16) into the 128B-swizzled
//              smem tile read by the A*V MMA.
//   warp 4*NG   TMEM allocator + TMA producer (lane 0): Q once, K/V ring.
//   warp 4*NG+1 MMA issuer (lane 0): S = Q K^T (TMEM, double buffered),
//              O += A V (TMEM accumulator, no rescaling — stick-breaking
//              weights are absolute).
#include "sb_args.cuh"

namespace sb {

template <int D, int NG>
struct FwdCfg {
  static constexpr int kStages = D == 128 ? 3 : 4;
  static constexpr int kCG = kBlock / NG;             // key columns per group
  static constexpr int kStick = 128 * NG;             // stick threads
  static constexpr int kThreads = kStick + 64;
  static constexpr int kQBytes = kTileM * D * 2;      // 128 x D bf16
  static constexpr int kKVBytes = kBlock * D * 2;     // 64 x D bf16
  static constexpr int kPBytes = kTileM * kBlock * 2; // 128 x 64 bf16
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKVBytes;
  static constexpr int kOffP = kOffV + kStages * kKVBytes;
  static constexpr int kOffX = kOffP + 2 * kPBytes;         // [2][NG][128] f32x2 partials
  static constexpr int kOffRed = kOffX + 2 * NG * 128 * 8;  // [2][4] f64 per-warp max(a)
  static constexpr int kOffBar = kOffRed + 2 * 4 * 8;
  static constexpr int kNumBars = 1 + 3 * kStages + 2 + 2 + 2 + 2 + 1;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = 256;           // S[2] (2x64) + O (D <= 128)
  static constexpr uint32_t kColS = 0, kColO = 128;
};

template <int D, int NG, bool kSkip>
__global__ void __launch_bounds__(FwdCfg<D, NG>::kThreads, 1)
    sb_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const FwdArgs args) {
  using C = FwdCfg<D, NG>;
  constexpr int ST = C::kStages;
  constexpr int CG = C::kCG;
  constexpr int kProdWarp = 4 * NG, kMmaWarp = 4 * NG + 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // heavy-first schedule: the last query tiles have the longest key sweeps
  const int BH = g.B * g.H;
  int item, bh;
  grouped_order((int)blockIdx.x, g.n_qt, BH, g.ugroup, item, bh);
  const int b = bh / g.H, h = bh % g.H;
  const Unit u = make_unit(g, b, h);
  if (item >= u.n_qt) return;  // shorter sequence of a varlen batch: no work
  const int qt = u.n_qt - 1 - item;
  const int qb0 = 2 * qt;
  const int kb_hi = min(qb0 + 1, u.nb - 1);  // diagonal block of the upper (or only) half
  const int n_kv = kb_hi + 1;                // tiles without skipping (kb = kb_hi .. 0)

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_vfull = bar_kfull + ST;
  uint64_t* bar_kvempty = bar_vfull + ST;
  uint64_t* bar_sfull = bar_kvempty + ST;
  uint64_t* bar_sempty = bar_sfull + 2;
  uint64_t* bar_pfull = bar_sempty + 2;
  uint64_t* bar_pempty = bar_pfull + 2;
  uint64_t* bar_ofull = bar_pempty + 2;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  uint32_t* tmem_slot = misc;                                       // TMEM base address
  volatile int* n_eff = reinterpret_cast<volatile int*>(misc + 1);  // tiles the MMA consumes
  float2* xch = reinterpret_cast<float2*>(smem + C::kOffX);
  double* red = reinterpret_cast<double*>(smem + C::kOffRed);

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_kfull + s, 1);
      mbar_init(bar_vfull + s, 1);
      mbar_init(bar_kvempty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_sfull + s, 1);
      mbar_init(bar_sempty + s, C::kStick);
      mbar_init(bar_pfull + s, C::kStick);
      mbar_init(bar_pempty + s, 1);
    }
    mbar_init(bar_ofull, 1);
    *n_eff = n_kv;
    fence_mbar_init();
  }
  if (warp == kProdWarp) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == kProdWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      const int row0 = qt * kTileM;
      mbar_expect_tx(bar_q, C::kQBytes);
      for (int c = 0; c < D / 64; ++c)
        tma_load_4d(&tm_q, bar_q, smem + C::kOffQ + c * (kTileM * 128), c * 64, u.trow0 + row0, h,
                    u.tb);
      int issued = 0;
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % ST;
        if (j >= ST) {
          const uint32_t par = ((j / ST) - 1) & 1;
          bool stop = false;
          while (!mbar_try_wait(bar_kvempty + s, par)) {
            if (kSkip && *n_eff <= j) { stop = true; break; }
          }
          if (stop) break;
        }
        if (kSkip && *n_eff <= j) break;
        const int kb = kb_hi - j;
        mbar_expect_tx(bar_kfull + s, C::kKVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_k, bar_kfull + s, smem + C::kOffK + s * C::kKVBytes + c * (kBlock * 128),
                      c * 64, u.trow0 + kb * kBlock, h, u.tb);
        mbar_expect_tx(bar_vfull + s, C::kKVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_v, bar_vfull + s, smem + C::kOffV + s * C::kKVBytes + c * (kBlock * 128),
                      c * 64, u.trow0 + kb * kBlock, h, u.tb);
        ++issued;
      }
      // never leave the CTA with bulk copies in flight (early exit under skip)
      for (int j = max(0, issued - ST); j < issued; ++j) {
        mbar_wait(bar_kfull + (j % ST), (j / ST) & 1);
        mbar_wait(bar_vfull + (j % ST), (j / ST) & 1);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T: both K-major
      constexpr uint32_t idesc_o = idesc_bf16(128, D, 0, 1);   // A V: V is MN-major
      const uint64_t dq = sdesc_sw128(smem_u32(smem + C::kOffQ), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(smem + C::kOffK), 16, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(smem + C::kOffV), kBlock * 128, 1024);
      const uint64_t dp = sdesc_sw128(smem_u32(smem + C::kOffP), 16, 1024);
      mbar_wait(bar_q, 0);
      auto issue_pv = [&](int i) -> bool {
        mbar_wait(bar_pfull + (i & 1), (i >> 1) & 1);
        const bool last = (*n_eff <= i + 1);
        const int s = i % ST;
        mbar_wait(bar_vfull + s, (i / ST) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kBlock / 16; ++k) {
          const uint64_t ad = desc_add(dp, (i & 1) * C::kPBytes + k * 32);
          const uint64_t bd = desc_add(dv, s * C::kKVBytes + k * 2048);
          umma_ss(tbase + C::kColO, ad, bd, idesc_o, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(bar_pempty + (i & 1));
        umma_commit(bar_kvempty + s);
        return last;
      };
      bool done = false;
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % ST;
        // K_j, unless the stick warps have already ended the sweep before tile j
        bool have_k = true;
        while (!mbar_try_wait(bar_kfull + s, (j / ST) & 1)) {
          if (kSkip && *n_eff <= j) { have_k = false; break; }
        }
        if (have_k) {
          if (j >= 2) mbar_wait(bar_sempty + (j & 1), ((j >> 1) + 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
            const uint64_t ad = desc_add(dq, off);
            const uint64_t bd = desc_add(dk, s * C::kKVBytes + offk);
            umma_ss(tbase + C::kColS + (j & 1) * 64, ad, bd, idesc_s, k > 0 ? 1u : 0u);
          }
          umma_commit(bar_sfull + (j & 1));
        }
        if (j >= 1) {
          done = issue_pv(j - 1);
          if (done) break;
        }
      }
      if (!done) issue_pv(n_kv - 1);
      umma_commit(bar_ofull);
    }
  } else {
    // ------------------------------------------------------------ stick warps
    const int quarter = warp & 3, gi = warp >> 2;  // row quarter, column group
    const int r = quarter * 32 + lane;             // TMEM lane == query row in the tile
    const int half = r >> 6;
    const int my_qb = qb0 + half;
    const int row = qt * kTileM + r;
    const bool row_valid = row < u.L;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    float* Mrow = args.M ? args.M + u.m_off + (r & 63) : nullptr;
    const uint32_t p_row = smem_u32(smem + C::kOffP) + r * 128;
    const int c0 = gi * CG;  // first key column of this group

    double a_d = 0.0;      // running log remaining mass (natural log), f64
    float a2 = 0.0f;       // same in log2 units, f32, feeds the exponent
    bool act[2] = {qb0 < u.nb, qb0 + 1 < u.nb};  // halves still sweeping
    int lowest = my_qb;    // leftmost processed key block (first_kb)
    int visited = 0;
    for (int j = 0; j < n_kv; ++j) {
      const int kb = kb_hi - j;
      const int par = j & 1;
      mbar_wait(bar_sfull + par, (j >> 1) & 1);
      tc_fence_after();
      float zs[CG];
      if constexpr (CG == 16) {
        tmem_ld16(tbase + lane_base + C::kColS + par * 64 + c0, zs);
      } else {
        tmem_ld32(tbase + lane_base + C::kColS + par * 64 + c0, zs);
      }
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar_sempty + par);

      // pass 1 over this group's columns (right to left). Exact skip path: log
      // space, exchange the group's sum of lt. Otherwise: product form, exchange
      // the group's product of r = exp(lt) and its log2.
      const bool mine = act[half] && kb <= my_qb;
      const bool diag = kb == my_qb;  // warp-uniform: a warp's rows share one half
      const int lim = diag ? (r & 63) : kBlock;  // strict causality on the diagonal
      float w[CG];
      float e1 = kSkip ? 0.0f : 1.0f, e2 = 0.0f;
      if (mine) {
        if constexpr (kSkip) {
          e1 = diag ? log_pass<CG, true>(zs, w, g.scale_log2, c0, lim)
                    : log_pass<CG, false>(zs, w, g.scale_log2, c0, lim);
        } else {
          if (diag) {
            e1 = prod_pass<CG, true>(zs, w, nullptr, g.scale_log2, c0, lim);
            e2 = group_log2<CG, true>(e1, zs, c0, lim);
          } else {
            e1 = prod_pass<CG, false>(zs, w, nullptr, g.scale_log2, c0, lim);
            e2 = group_log2<CG, false>(e1, zs, c0, lim);
          }
        }
      }
      xch[(par * NG + gi) * 128 + r] = make_float2(e1, e2);
      if (kSkip && gi == 0 && j > 0) {
        // skip check for this tile (blocked.py:175-176), on a after the previous one
        double m = row_valid ? a_d : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) red[par * 4 + quarter] = m;
      }
      named_bar_sync(1, C::kStick);
      if (kSkip && j > 0) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const double mh = fmax(red[par * 4 + 2 * hh], red[par * 4 + 2 * hh + 1]);
          if (act[hh] && kb < qb0 + hh && mh < args.log_eps) act[hh] = false;
        }
      }
      const bool live = act[half] && kb <= my_qb;
      // right: what the groups right of mine contribute; tot: the whole row's lt (log2)
      float right = kSkip ? 0.0f : 1.0f, tot = 0.0f;
#pragma unroll
      for (int g2 = 0; g2 < NG; ++g2) {
        const float2 v = xch[(par * NG + g2) * 128 + r];
        if (kSkip) {
          tot += v.x;
          if (g2 > gi) right += v.x;
        } else {
          tot += v.y;
          if (g2 > gi) right *= v.x;
        }
      }
      uint32_t pk[CG / 2];
      if (live) {
        if constexpr (kSkip) {
          const float base = right + a2;
#pragma unroll
          for (int c = 0; c < CG; c += 2) {
            const float A0 = (!diag || c0 + c < lim) ? ex2(zs[c] + w[c] + base) : 0.0f;
            const float A1 = (!diag || c0 + c + 1 < lim) ? ex2(zs[c + 1] + w[c + 1] + base) : 0.0f;
            pk[c >> 1] = pack_bf16(A0, A1);
          }
        } else {
          const float base = ex2(a2) * right;
#pragma unroll
          for (int c = 0; c < CG; c += 2) pk[c >> 1] = pack_bf16(w[c] * base, w[c + 1] * base);
        }
        if (gi == 0 && Mrow && row_valid) Mrow[tile_index(my_qb, kb) * kBlock] = a2;
        a_d += (double)tot * (double)kLn2;
        a2 = (float)(a_d * 1.4426950408889634);
        lowest = kb;
        ++visited;
      } else {
#pragma unroll
        for (int c = 0; c < CG / 2; ++c) pk[c] = 0u;
      }
      const bool stop = kSkip && !act[0] && !act[1];
      if (stop && r == 0 && gi == 0) *n_eff = j + 1;  // tile j (all-zero A) is the last one
      if (j >= 2) mbar_wait(bar_pempty + par, ((j >> 1) + 1) & 1);
      const uint32_t pb = p_row + par * C::kPBytes;
#pragma unroll
      for (int c = 0; c < CG / 8; ++c) {
        const int chunk = gi * (CG / 8) + c;
        st_shared_v4(pb + ((chunk ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                     pk[4 * c + 3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(bar_pfull + par);
      if (stop) break;
    }

    // ------------------------------------------------------------ epilogue
    mbar_wait(bar_ofull, 0);
    tc_fence_after();
    constexpr int DC = D / NG;  // output columns per group (16 or 32)
    float ov[DC];
    if constexpr (DC == 16) {
      tmem_ld16(tbase + lane_base + C::kColO + gi * DC, ov);
    } else {
      tmem_ld32(tbase + lane_base + C::kColO + gi * DC, ov);
    }
    tmem_wait_ld();
    if (row_valid) {
      __nv_bfloat16* orow = args.o + u.out_off + (int64_t)row * g.sl + gi * DC;
      uint4* dst = reinterpret_cast<uint4*>(orow);
#pragma unroll
      for (int q4 = 0; q4 < DC / 8; ++q4)
        dst[q4] = make_uint4(pack_bf16(ov[8 * q4], ov[8 * q4 + 1]),
                             pack_bf16(ov[8 * q4 + 2], ov[8 * q4 + 3]),
                             pack_bf16(ov[8 * q4 + 4], ov[8 * q4 + 5]),
                             pack_bf16(ov[8 * q4 + 6], ov[8 * q4 + 7]));
      if (gi == 0) args.log_rem[u.rem_off + row * u.rem_stride] = (float)a_d;
    }
    if (gi == 0 && my_qb < u.nb && (r & 63) == 0) {
      args.first_kb[u.fkb_off + my_qb] = lowest;
      if (args.counters) atomicAdd(args.counters, (unsigned long long)visited);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProdWarp) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D, int NG, bool kSkip>
static int launch_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      const FwdArgs& a, cudaStream_t stream) {
  using C = FwdCfg<D, NG>;
  auto kern = sb_fwd_kernel<D, NG, kSkip>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  if (e != cudaSuccess) return (int)e;
  const unsigned grid = (unsigned)(a.g.n_qt * a.g.B * a.g.H);
  kern<<<grid, C::kThreads, C::kSmem, stream>>>(tq, tk, tv, a);
  return (int)cudaGetLastError();
}

constexpr int kFwdGroups = 4;

int fwd_dispatch(int D, bool skip, const CUtensorMap& tq, const CUtensorMap& tk,
                 const CUtensorMap& tv, const FwdArgs& a, cudaStream_t stream) {
  if (D == 128) return skip ? launch_fwd<128, kFwdGroups, true>(tq, tk, tv, a, stream)
                            : launch_fwd<128, kFwdGroups, false>(tq, tk, tv, a, stream);
  if (D == 64) return skip ? launch_fwd<64, kFwdGroups, true>(tq, tk, tv, a, stream)
                           : launch_fwd<64, kFwdGroups, false>(tq, tk, tv, a, stream);
  return -1;
}

}  // namespace sb
